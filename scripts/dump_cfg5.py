"""Dump the cfg5 col_idx (int32) for scripts/probe_gather.cu (investigation only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
g = synth.cfg5()
g["col_idx"].astype("int32").tofile(sys.argv[1] if len(sys.argv) > 1 else "/tmp/cfg5_col.bin")
print("nnz", g["col_idx"].size)
