// status.cuh -- ilans_status helpers shared by the extern "C" entry points.
#pragma once

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

// ---------------------------------------------------------------------------
// status helpers
// ---------------------------------------------------------------------------
inline void st_clear(ilans_status *st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->stream = -1;
    st->index = -1;
    st->symbol = -1;
}

inline int st_fail(ilans_status *st, int code, const char *fmt, ...) {
    if (st) {
        st->code = code;
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(st->message, sizeof(st->message), fmt, ap);
        va_end(ap);
    }
    return code;
}

inline int st_cuda(ilans_status *st, cudaError_t e, const char *where) {
    if (st) st->cuda_error = static_cast<int32_t>(e);
    return st_fail(st, ILANS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return st_cuda(st, _e, #expr); \
    } while (0)


// The calling host thread's device context (capi.cu): selects the device,
// locks its context and returns the library stream the call runs on.
int ilans_host_session(ilans_status *st, cudaStream_t *stream, std::unique_lock<std::mutex> *lock);
