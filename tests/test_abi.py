"""Host-side checks of the C ABI (no GPU, no compute): the library builds/loads, exports every
symbol include/mapi.h declares, validates arguments before touching the device, and its MAVP
inner loops contain no multiplication (SASS inspection, the analogue of the paper's op-count
claim P:5 / P:146)."""
import ctypes
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

import paper_2110_12065_b200 as m

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mapi.h")


@pytest.fixture(scope="module")
def lib():
    m.build()
    return m.load()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mapi_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 13
    for name in names:
        assert hasattr(lib, name), f"{name} declared in mapi.h but not exported"
    out = subprocess.run(["nm", "-D", "--defined-only", m._build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mapi_\w+)", out))
    assert set(names) <= exported


def test_status_strings(lib):
    for code, name in m.STATUS.items():
        assert lib.mapi_status_string(code).decode() == name


def test_workspace_sizes_monotone(lib):
    a = m.workspace_size(m.WS_ITERATE, 1000)
    b = m.workspace_size(m.WS_ITERATE, 2000)
    assert 0 < a < b
    assert m.workspace_size(m.WS_MATVEC, 1000) == 0
    assert m.workspace_size(m.WS_ITERATE_HOST, 100, 104, 50) >= 100 * 104 * 4
    assert m.workspace_size(m.WS_PCA_TOPK, 64, 0, 8) >= 64 * 64 * 4
    assert m.workspace_size(m.WS_RANK_CSR, 1000, 5000) > 0
    assert m.workspace_size(m.WS_ITERATE_BATCHED, 1000, 0, 64) >= 2 * 64 * 1000 * 4


def _err(lib):
    return lib.mapi_last_error_message().decode()


def test_validation_before_device(lib):
    # every one of these fails argument validation on the host, before any CUDA call
    fake = ctypes.c_void_p(4096)  # never dereferenced
    st = lib.mapi_iterate(0, None, 4, 4, fake, 5, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 1 and "A is NULL" in _err(lib)
    st = lib.mapi_iterate(0, fake, 4, 3, fake, 5, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 2 and "lda (3) < n (4)" in _err(lib)
    st = lib.mapi_iterate(0, fake, 4, 4, fake, 0, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 3 and "iters" in _err(lib)
    st = lib.mapi_iterate(0, fake, 4, 4, fake, 5, -1.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 3 and "tol" in _err(lib)
    st = lib.mapi_iterate(7, fake, 4, 4, fake, 5, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 3 and "op" in _err(lib)
    st = lib.mapi_iterate(0, fake, 4, 4, fake, 5, 0.0, fake, None, None, None, None, fake, 16, None)
    assert st == 7
    # the symmetric entry point validates the same way; its workspace adds the K2s partial buffers
    st = lib.mapi_iterate_sym(0, None, 4, 4, fake, 5, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 1 and "A is NULL" in _err(lib)
    st = lib.mapi_iterate_sym(0, fake, 4, 3, fake, 5, 0.0, fake, None, None, None, None, fake, 1 << 20, None)
    assert st == 2 and "lda (3) < n (4)" in _err(lib)
    st = lib.mapi_iterate_sym(0, fake, 4, 4, fake, 5, 0.0, fake, None, None, None, None, fake, 16, None)
    assert st == 7
    n = 32768
    assert m.workspace_size(m.WS_ITERATE_SYM, n) == m.workspace_size(m.WS_ITERATE, n) + \
        4 * n * (n // 128 + n // 256)
    st = lib.mapi_mavp_matvec(0, fake, 3, 10, 9, fake, fake, None)
    assert st == 2 and "lda (9) < n_cols (10)" in _err(lib)
    st = lib.mapi_pca_topk(0, fake, 8, 8, 9, 5, fake, fake, None, None, fake, 1 << 30, None)
    assert st == 3 and "k (9)" in _err(lib)
    st = lib.mapi_csr_prepare(10, 5, fake, fake, 1.5, fake, fake, fake, 1 << 20, None)
    assert st == 3 and "alpha" in _err(lib)
    st = lib.mapi_rank_csr(10, 5, fake, fake, fake, fake, fake, 0, 0.0, fake, None, None, None, fake,
                           1 << 20, None)
    assert st == 3 and "max_iters" in _err(lib)
    st = lib.mapi_iterate_batched(0, fake, 8, 8, fake, 0, 5, 0.0, fake, None, None, None, fake, 1 << 30, None)
    assert st == 3 and "k (0)" in _err(lib)
    # fused P2P sharding (K2p): argument checks before any CUDA call
    sh = lambda **kw: lib.mapi_iterate_sharded(  # noqa: E731
        kw.get("op", 0), kw.get("A", fake), kw.get("m", 256), kw.get("n", 512), kw.get("lda", 512),
        kw.get("row0", 0), fake, kw.get("iters", 5), kw.get("tol", 0.0), kw.get("rank", 0), kw.get("world", 2),
        kw.get("peers", fake), 0, 0, kw.get("grid", 8), fake, None, None, None, None, None, fake,
        kw.get("ws_bytes", 1 << 20), None)
    assert sh(peers=None) == 1 and "NULL" in _err(lib)
    assert sh(world=0) == 3 and "world" in _err(lib)
    assert sh(rank=2) == 3 and "rank 2" in _err(lib)
    assert sh(n=128, m=64, lda=128) == 2 and "n >= 256" in _err(lib)
    assert sh(row0=300) == 2
    assert sh(lda=516) == 2 and "32 B-aligned" in _err(lib)
    assert sh(iters=0) == 3 and "iters" in _err(lib)
    assert sh(ws_bytes=16) == 7
    assert sh(op=5) == 3
    assert sh(grid=0) == 3 and "explicit grid" in _err(lib)  # world > 1 must pass the agreed grid
    assert sh(grid=5000) == 3
    # sharded symmetric (K2sp): the held rows must be the shard's, before any CUDA call
    ssh = lambda **kw: lib.mapi_iterate_sym_sharded(  # noqa: E731
        0, fake, kw.get("lo", 0), kw.get("hi", 1), kw.get("n", 8192), 8192, fake, 5, 0.0, kw.get("rank", 0),
        kw.get("world", 2), fake, 0, 0, 8, fake, None, None, None, None, None, fake, 1 << 30, None)
    assert ssh() == 2 and "mapi_sym_shard_rows" in _err(lib)
    assert ssh(n=1001) == 2
    assert ssh(world=0) == 3
    # pipelined host problems
    arr = (ctypes.c_void_p * 1)(fake.value)
    st = lib.mapi_iterate_host_many(0, 0, arr, 4, 4, arr, 5, 0.0, arr, None, None, None, fake, 1 << 20, None)
    assert st == 3 and "count" in _err(lib)
    st = lib.mapi_iterate_host_many(0, 1, None, 4, 4, arr, 5, 0.0, arr, None, None, None, fake, 1 << 20, None)
    assert st == 1
    st = lib.mapi_iterate_host_many(0, 1, arr, 4, 4, arr, 5, 0.0, arr, None, None, None, fake, 16, None)
    assert st == 7
    # packed symmetric host problems: same validation (lda is derived from n)
    st = lib.mapi_iterate_host_many_packed(0, 0, arr, 4, arr, 5, 0.0, arr, None, None, None, fake, 1 << 20, None)
    assert st == 3 and "count" in _err(lib)
    st = lib.mapi_iterate_host_many_packed(0, 1, arr, 0, arr, 5, 0.0, arr, None, None, None, fake, 1 << 20, None)
    assert st == 2
    st = lib.mapi_iterate_host_many_packed(0, 1, arr, 4, arr, 5, 0.0, arr, None, None, None, fake, 16, None)
    assert st == 7
    assert m.workspace_size(m.WS_ITERATE_HOST_MANY_PACKED, 1000, 0, 50) >= \
        m.workspace_size(m.WS_ITERATE_HOST_MANY, 1000, 1000, 50) + 2 * 4 * 1000 * 1001 // 2


def test_csr_reorder_permute_validation(lib):
    """mapi_csr_reorder / mapi_csr_permute validate on the host before touching the device."""
    fake = ctypes.c_void_p(4096)
    ws = m.workspace_size(m.WS_CSR_REORDER, 1000)
    assert ws > 5 * 4 * 1000
    st = lib.mapi_csr_reorder(0, 10, fake, fake, fake, fake, fake, fake, ws, None)
    assert st == 2
    st = lib.mapi_csr_reorder(1000, 10, None, fake, fake, fake, fake, fake, ws, None)
    assert st == 1
    st = lib.mapi_csr_reorder(1000, 10, fake, fake, fake, fake, fake, fake, 16, None)
    assert st == 7
    st = lib.mapi_csr_reorder(1000, 1 << 40, fake, fake, fake, fake, fake, fake, ws, None)
    assert st == 2 and "int32" in _err(lib)
    # the same bounds as mapi_csr_prepare / mapi_rank_csr: n + 1 and nnz must fit the int32 scan
    big = (1 << 31) - 1
    assert lib.mapi_csr_reorder(big, 10, fake, fake, fake, fake, fake, fake, 1 << 62, None) == 2
    assert lib.mapi_csr_reorder(1000, big, fake, fake, fake, fake, fake, fake, ws, None) == 2
    assert lib.mapi_csr_permute(0, fake, fake, fake, 1, None) == 2
    assert lib.mapi_csr_permute(10, None, fake, fake, 1, None) == 1
    assert lib.mapi_csr_permute(10, fake, fake, fake, 1, None) == 3  # x aliases out


def test_rank_csr_shard_validation(lib):
    """mapi_rank_csr_shard_* (K3n) validate on the host before touching the device; the workspace grows with the
    node count (full node state on every rank) and with the rank's rows + edges (merge-path tiles)."""
    fake = ctypes.c_void_p(4096)
    n, m_rows, nnz = 1000, 300, 5000
    ws = m.workspace_size(m.WS_RANK_CSR_SHARD, n, nnz, m_rows)
    assert ws >= 256 + 3 * 4 * n
    assert m.workspace_size(m.WS_RANK_CSR_SHARD, 2 * n, nnz, m_rows) > ws
    assert m.workspace_size(m.WS_RANK_CSR_SHARD, n, 100 * nnz, m_rows) > ws
    assert m.workspace_size(m.WS_RANK_CSR_SHARD, n, nnz, n) <= m.workspace_size(m.WS_RANK_CSR, n, nnz)
    begin, rows, norm, fin = (lib.mapi_rank_csr_shard_begin, lib.mapi_rank_csr_shard_rows,
                              lib.mapi_rank_csr_shard_normalize, lib.mapi_rank_csr_shard_finish)
    assert begin(0, 0, 0, fake, fake, fake, fake, fake, ws, None) == 2
    assert begin(n, n + 1, nnz, fake, fake, fake, fake, fake, 1 << 40, None) == 2 and "rows" in _err(lib)
    assert begin(n, m_rows, 1 << 40, fake, fake, fake, fake, fake, 1 << 60, None) == 2
    assert begin(n, m_rows, nnz, fake, fake, fake, fake, None, ws, None) == 7
    assert begin(n, m_rows, nnz, fake, fake, fake, fake, fake, 16, None) == 7
    assert begin(n, m_rows, nnz, None, fake, fake, fake, fake, ws, None) == 1
    assert begin(n, m_rows, nnz, fake, None, fake, fake, fake, ws, None) == 1
    assert rows(n, m_rows, 800, nnz, fake, fake, 0, None, fake, ws, None) == 2  # rows [800, 1100) leave [0, n)
    assert rows(n, m_rows, 0, nnz, fake, None, 0, None, fake, ws, None) == 1
    assert rows(n, m_rows, 0, nnz, fake, fake, -1, None, fake, ws, None) == 3
    assert norm(n, m_rows, nnz, fake, fake, None, 0, 0.0, None, fake, ws, None) == 1
    assert norm(n, m_rows, nnz, fake, fake, fake, 0, -1.0, None, fake, ws, None) == 3
    assert norm(n, m_rows, nnz, fake, fake, fake, -2, 0.0, None, fake, ws, None) == 3
    assert fin(n, m_rows, nnz, fake, fake, None, None, None, None, ws, None) == 7
    assert fin(n, m_rows, nnz, None, fake, None, None, None, fake, ws, None) == 1

def test_pack_upper_layout():
    """pack_upper: row j of the packed buffer is A[j, j:], rows back to back (offset j n - j (j-1) / 2),
    checked against numpy's triu index order on odd / even sizes."""
    for n in (1, 2, 7, 64, 101):
        A = np.arange(n * n, dtype=np.float32).reshape(n, n)
        got = m.pack_upper(A).numpy()
        iu = np.triu_indices(n)
        assert np.array_equal(got, A[iu])
        for j in (0, n // 2, n - 1):
            off = j * n - j * (j - 1) // 2
            assert np.array_equal(got[off:off + n - j], A[j, j:])


def test_p2p_exchange_layout_and_new_workspaces(lib):
    """Exchange buffer = 256 B flag header + y (fp32) for two parities x world source ranks + fp64 rank
    totals (2 x world); the K2p workspace holds its status header and the per-CTA partials (2 x 1024)."""
    al = lambda b: (b + 255) // 256 * 256  # noqa: E731
    for n, world in ((4096, 2), (32768, 8), (1000, 1)):
        assert lib.mapi_p2p_exchange_bytes(n, world) == 256 + al(8 * world * n) + al(16 * world)
    assert lib.mapi_p2p_exchange_bytes(100, 0) == 0
    assert lib.mapi_workspace_size(m.WS_ITERATE_SHARDED, 0, 0, 0) == 256 + 16 * 1024
    one = lib.mapi_workspace_size(m.WS_ITERATE_HOST, 1024, 1024, 50)
    many = lib.mapi_workspace_size(m.WS_ITERATE_HOST_MANY, 1024, 1024, 50)
    assert many > one and many >= 2 * 4 * 1024 * 1024  # two A slots


def _sass_functions():
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "-sass", m._build.LIB], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        mm = re.match(r"\s+Function : (\S+)", line)
        if mm:
            cur = mm.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


FMULS = re.compile(r"\b(FMUL|FFMA|DMUL|DFMA|HMUL2|HFMA2|FMUL2|FFMA2)\b")


def _blocks(lines):
    """Split a SASS listing into basic blocks at labels (.L_x_NN:) and branches."""
    block = []
    for ln in lines:
        if re.match(r"\s*\.L_\w+:", ln):
            if block:
                yield block
            block = []
            continue
        block.append(ln)
        if re.search(r"\b(BRA|EXIT|RET|BRX|CALL)\b", ln):
            yield block
            block = []
    if block:
        yield block


def _real_mul(ln):
    # `HFMA2 Rd, -RZ, RZ, imm` is ptxas' constant-materialisation idiom (0 * 0 + imm), not a multiply
    return bool(FMULS.search(ln)) and "-RZ, RZ," not in ln


def test_mavp_loops_have_no_multiply(lib):
    """AC3 analogue (P:5): no floating multiply in any basic block that evaluates MAVP terms
    (FMNMX.XORSIGN), in every MAVP kernel; the pure streaming mat-vec kernels have none at all (the
    iteration kernels' only multiplies are the Newton steps of the l1-normalisation divisions)."""
    funcs = _sass_functions()
    mavp = [f for f in funcs if any("FMNMX.XORSIGN" in ln for ln in funcs[f])]
    names = " ".join(mavp)
    for k in ("k_matvec", "k_rows_partial", "k_iterate_persistent", "k_iterate_coop", "k_batched_partial"):
        assert k in names, f"no FMNMX.XORSIGN kernel named {k}"
    for f in mavp:
        for blk in _blocks(funcs[f]):
            if any("FMNMX" in ln for ln in blk):
                bad = [ln.strip() for ln in blk if _real_mul(ln)]
                assert not bad, f"{f}: multiply in an MAVP block:\n" + "\n".join(bad[:4])
    # (the ILi2E instantiations are the RPI comparator, op = MAPI_OP_DOT: the regular product of Eq. 1)
    # (k_matvec_norm is excluded here: its prologue divides y by s; its MAVP blocks are checked above)
    streaming = [f for f in funcs if re.search(r"8k_matvecI|k_rows_partial|k_batched_partial|k_rank_rows", f)
                 and not re.search(r"k_(matvec|rows_partial|batched_partial)ILi2E", f)]
    assert len(streaming) >= 8
    for f in streaming:
        fmul = [ln for ln in funcs[f] if _real_mul(ln)]
        assert not fmul, f"{f} has floating multiplies:\n" + "\n".join(fmul[:5])


def test_streaming_loads_are_256bit(lib):
    funcs = _sass_functions()
    hits = [f for f in funcs if "k_iterate_persistentILi0ELi8ELi0" in f]
    assert hits
    body = "\n".join(funcs[hits[0]])
    assert re.search(r"LDG\.E\.NA\.EFL2\.256", body) or re.search(r"LDG\.E\.EF.*\.256", body), \
        "expected 256-bit evict-first streaming loads"
