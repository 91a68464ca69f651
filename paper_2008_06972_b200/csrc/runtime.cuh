// Host-side runtime helpers shared by the encoder and decoder contexts:
// grow-only device / pinned-host workspaces and the thread-local error text
// behind stpc_last_error().
#pragma once
#include <string>

#include <cuda_runtime.h>

#include "../../include/stpc_b200.h"

namespace stpc {

void set_last_error(const std::string& msg);

struct DevBuf;
#ifdef STPC_GUARD
// Write-guard build (tools/guard_check.py): the bytes of every workspace past
// the size its last ensure() asked for hold a canary, checked after each call
// by stpc_debug_guard_check -- an out-of-bounds write of any kernel into its
// own buffer's slack shows up as a changed canary.  (compute-sanitizer is not
// available on the GPU pool.)
void guard_arm(DevBuf* b, size_t from);
void guard_forget(DevBuf* b);
#endif

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    size_t used = 0;  // bytes the last ensure() asked for
    int ensure(size_t need)
    {
        if (need <= cap) {
#ifdef STPC_GUARD
            if (need != used) guard_arm(this, need);
#endif
            used = need;
            return 0;
        }
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t c = need + need / 8 + 256;
        if (cudaMalloc(&p, c) != cudaSuccess) {
            set_last_error("cudaMalloc failed (" + std::to_string(c) + " bytes)");
            return STPC_ERR_NOMEM;
        }
        cap = c;
        used = need;
#ifdef STPC_GUARD
        guard_arm(this, need);
#endif
        return 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf()
    {
#ifdef STPC_GUARD
        guard_forget(this);
#endif
        if (p) cudaFree(p);
    }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    int ensure(size_t need)
    {
        if (need <= cap) return 0;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t c = need + need / 8 + 256;
        if (cudaMallocHost(&p, c) != cudaSuccess) {
            set_last_error("cudaMallocHost failed");
            return STPC_ERR_NOMEM;
        }
        cap = c;
        return 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
    ~HostBuf()
    {
        if (p) cudaFreeHost(p);
    }
};


}  // namespace stpc
