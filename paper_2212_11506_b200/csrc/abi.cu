// Error slot and version of the C ABI (include/bhtsne_b200.h).
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace bh {

static thread_local char g_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return BH_OK;
    return set_error(BH_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace bh

extern "C" const char *bh_last_error(void) { return bh::g_err; }

extern "C" int bh_abi_version(void) { return BH_ABI_VERSION; }

extern "C" int64_t bh_tree_node_bound(int64_t n, int code_bits) {
    // every sorted point starts nodes on at most max_depth + 1 levels
    return n * (int64_t)(code_bits / 2 + 1) + 1;
}
