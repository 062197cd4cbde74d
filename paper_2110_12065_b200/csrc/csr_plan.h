// csr_plan.h — sizes of the segmented CSR ranking path (K3s, csr_plan.cu), for mapi_workspace_size.
#pragma once
#include <cstddef>
#include <cstdint>

namespace mapi_plan {
size_t plan_bytes_bound(int64_t n, int64_t nnz);   // the plan buffer (upper bound before the build)
size_t plan_build_ws_bytes(int64_t n, int64_t nnz);  // temporary workspace of mapi_csr_plan
size_t rank_plan_ws_bytes(int64_t n, int64_t nnz);   // workspace of mapi_rank_csr_plan
}  // namespace mapi_plan
