// hp_common.cuh — shared helpers for the HashPoint sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/hashpoint_b200.h"

namespace hp {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
void count_launch(int n = 1);

// Optional per-kernel CUDA-event timing (hp_timing_enable): spans recorded on
// the launching stream around the named launches, summed per name.
void timing_begin(const char* name, cudaStream_t s);
void timing_end(cudaStream_t s);
struct TimedSpan {
    cudaStream_t s;
    TimedSpan(const char* name, cudaStream_t st) : s(st) { timing_begin(name, st); }
    ~TimedSpan() { timing_end(s); }
};

#define HP_CHECK_LAUNCH(where)                                                 \
    do {                                                                       \
        ::hp::count_launch();                                                  \
        cudaError_t _e = cudaGetLastError();                                   \
        if (_e != cudaSuccess) return ::hp::cuda_status(_e, where);            \
    } while (0)

// ---------------------------------------------------------------- checked build
// `make checked` (-DHP_CHECKED) builds libhp_b200_checked.so: HP_ASSERT
// records the first failing check of each translation unit (source line)
// in a device word instead of touching memory out of bounds;
// hp_check_failures() reads them (the test suite runs against it: the
// substitute for compute-sanitizer, which is closed on this pool).  In the
// normal build HP_ASSERT compiles to nothing.
using CheckReader = int (*)(unsigned long long* out, int reset);
int register_check_reader(CheckReader f);
#ifdef HP_CHECKED
static __device__ unsigned long long g_hp_check;
#define HP_ASSERT(c)                                                                     \
    do {                                                                                 \
        if (!(c)) atomicCAS(&::hp::g_hp_check, 0ull, (unsigned long long)__LINE__);      \
    } while (0)
namespace {
[[maybe_unused]] const int hp_check_registered = register_check_reader([](unsigned long long* out, int reset) -> int {
    if (cudaMemcpyFromSymbol(out, g_hp_check, sizeof(*out)) != cudaSuccess) return -1;
    if (reset) {
        const unsigned long long z = 0;
        if (cudaMemcpyToSymbol(g_hp_check, &z, sizeof(z)) != cudaSuccess) return -1;
    }
    return 0;
});
}  // namespace
#else
#define HP_ASSERT(c) ((void)0)
#endif

#define HP_TRY(expr)                                                           \
    do {                                                                       \
        int _rc = (expr);                                                      \
        if (_rc != HP_OK) return _rc;                                          \
    } while (0)

// SM count of the current device (148 on a B200: 2 dies x 74), cached per device
int device_sms();
// Resident CTAs per SM of `fn` at this block size / dynamic shared memory on
// the current device; sets the kernel's max-dynamic-shared-memory attribute
// there first (once per device).  Negative HP_E* on failure.
int kernel_occupancy(const void* fn, int threads, size_t smem);

// ---------------------------------------------------------------- workspace
// Bump allocator over the caller's workspace; every carve is 256-B aligned.
struct Carver {
    char* base;
    size_t cap;
    size_t used = 0;
    Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <class T>
    T* take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        used = off + count * sizeof(T);
        return reinterpret_cast<T*>(base ? base + off : nullptr);
    }
    bool ok() const { return used <= cap; }
};

// ---------------------------------------------------------------- fp64, no FMA
// The reference (numba, fastmath off) evaluates left to right without
// contraction.  The library is compiled with -fmad=false; these wrappers make
// the intent explicit at the parity-critical sites.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// Monotone key of a double: unsigned order == numeric order (no NaN).
__device__ __forceinline__ unsigned long long okey(double x) {
    unsigned long long b = __double_as_longlong(x);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Dynamic work distribution for warp-per-item kernels: lane 0 claims kBatch
// items at a time from a zeroed global counter (item costs vary widely, so a
// static split leaves a long tail).  Warp-uniform.
template <int kBatch>
struct WarpClaim {
    unsigned long long* ctr;
    int64_t cur = 0, end = 0;
    __device__ __forceinline__ explicit WarpClaim(unsigned long long* c) : ctr(c) {}
    __device__ __forceinline__ bool next(int64_t n, int64_t& item) {
        if (cur >= end) {
            unsigned long long b = 0;
            if ((threadIdx.x & 31) == 0) b = atomicAdd(ctr, (unsigned long long)kBatch);
            b = __shfl_sync(0xffffffffu, b, 0);
            cur = int64_t(b);
            end = cur + kBatch;
        }
        if (cur >= n) return false;
        item = cur++;
        return true;
    }
};
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// inclusive warp scan
template <class T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane_id() >= o) v += u;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns the exclusive
// prefix, writes the block total to *total.  `sh` needs blockDim/32 + 1 slots.
// kTail = false: no trailing barrier (the caller syncs before `sh` is reused).
template <class T, bool kTail = true>
__device__ __forceinline__ T block_excl_scan(T v, T* sh, T* total) {
    const int nw = blockDim.x >> 5;
    T inc = warp_incl_scan(v);
    if (lane_id() == 31) sh[warp_id()] = inc;
    __syncthreads();
    if (warp_id() == 0) {
        T w = lane_id() < nw ? sh[lane_id()] : T(0);
        T wi = warp_incl_scan(w);
        if (lane_id() < nw) sh[lane_id()] = wi - w;
        if (lane_id() == nw - 1) sh[nw] = wi;
    }
    __syncthreads();
    T res = inc - v + sh[warp_id()];
    *total = sh[nw];
    if (kTail) __syncthreads();
    return res;
}

inline unsigned grid_for(int64_t n, int threads, int64_t cap = 148 * 64) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return static_cast<unsigned>(g);
}

// ---------------------------------------------------------------- device scan
// Exclusive scan of `n` int64 (or int32 widened) values into int64 out[n+1]
// (out[n] = total).  In-place allowed.  Workspace: scan_workspace_bytes(n).
size_t scan_workspace_bytes(int64_t n);
int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t s);
int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t s);
int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, void* ws,
                              cudaStream_t s);

// cp.async (LDGSTS) helpers: asynchronous global -> shared copies.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace hp
