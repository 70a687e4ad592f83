// Error reporting and launch accounting shared by every entry point.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace fscnn {

namespace {
thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return FSCNN_ERR_CUDA;
    }
    note_launch(1);
    return FSCNN_OK;
}

}  // namespace fscnn

extern "C" {

int fscnn_abi_version(void) { return 1; }

const char *fscnn_last_error(void) { return fscnn::g_err; }

int64_t fscnn_launch_count(void) { return fscnn::g_launches.load(); }

void fscnn_reset_launch_count(void) { fscnn::g_launches.store(0); }

void fscnn_add_launch_count(int64_t n) { fscnn::g_launches.fetch_add(n); }

}  // extern "C"
