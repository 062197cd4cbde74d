// minibatch.h — sizes of the mini-batch MAPI path (K10, minibatch.cu), for mapi_workspace_size.
#pragma once
#include <cstddef>
#include <cstdint>

namespace mapi_mb {
size_t minibatch_ws_bytes(int64_t D, int64_t s, int64_t T);  // workspace of mapi_minibatch
}  // namespace mapi_mb
