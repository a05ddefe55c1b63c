// hp_query_core.cuh — pieces shared by the query kernels (hp_query.cu: full
// CSR; hp_head.cu: sample-only heads): ray groups, the row-major footprint
// tabulation, order keys, the exact (t, id) ranking of a staged segment.
#pragma once

#include <math_constants.h>

#include <cfloat>
#include <climits>

#include "hp_common.cuh"
#include "hp_cone.cuh"

namespace hp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroupMax = 32;  // rays per group

struct Rays {
    const int64_t* pix;
    int64_t pstride;
    const double* dirs;
    const double* tn;
    const double* tf;
    const double* slopes;
};

__device__ __forceinline__ RayParams load_ray(const Rays& R, int64_t r) {
    RayParams p;
    p.u = int(R.pix[r * R.pstride]);
    p.v = int(R.pix[r * R.pstride + 1]);
    p.d0 = R.dirs[3 * r];
    p.d1 = R.dirs[3 * r + 1];
    p.d2 = R.dirs[3 * r + 2];
    p.tn = R.tn[r];
    p.tf = R.tf[r];
    p.slope = R.slopes[r];
    ray_derive(p);
    return p;
}

constexpr int kRowsMax = 48;  // kernel rows tabulated per batch

struct GroupHead {
    RayParams ray[kGroupMax];
    Footprint fp[kGroupMax];
    int rlo[kRowsMax][kGroupMax], rhi[kRowsMax][kGroupMax];  // ray's tested sub-range per row
    int slo[kRowsMax], shi[kRowsMax];                          // staged (union) range per row
    int u0, u1, v0, v1;
};

struct QCam {  // camera frame for the footprint (has_cam == 0: full windows)
    CamFrame C;
    int has_cam, width, height;
};

// Group bounding box (padded coordinates) of rays [r0, r0+G).
__device__ void group_setup(GroupHead& S, const Rays& R, const QCam& QC, int64_t r0, int G, int s) {
    const int tid = threadIdx.x;
    if (tid < G) {
        S.ray[tid] = load_ray(R, r0 + tid);
        if (QC.has_cam)
            footprint_init(S.fp[tid], QC.C, S.ray[tid].d0, S.ray[tid].d1, S.ray[tid].d2, S.ray[tid].slope);
        else
            S.fp[tid].tight = 0;
    }
    __syncthreads();
    if (tid < 32) {
        int u0 = INT_MAX, u1 = INT_MIN, v0 = INT_MAX, v1 = INT_MIN;
        if (tid < G) {
            u0 = S.ray[tid].u;
            u1 = S.ray[tid].u + s;
            v0 = S.ray[tid].v;
            v1 = S.ray[tid].v + s;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            u0 = min(u0, __shfl_xor_sync(0xffffffffu, u0, o));
            u1 = max(u1, __shfl_xor_sync(0xffffffffu, u1, o));
            v0 = min(v0, __shfl_xor_sync(0xffffffffu, v0, o));
            v1 = max(v1, __shfl_xor_sync(0xffffffffu, v1, o));
        }
        if (tid == 0) {
            S.u0 = u0;
            S.u1 = u1;
            S.v0 = v0;
            S.v1 = v1;
        }
    }
    __syncthreads();
}

// Order-preserving uint32 key of a float (and back).
__device__ __forceinline__ unsigned fkey(float x) {
    const unsigned u = __float_as_uint(x);
    return u ^ (unsigned(int(u) >> 31) | 0x80000000u);  // negative: all bits flipped; else the sign bit
}
__device__ __forceinline__ float from_fkey(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ bool key_less(double ta, int64_t ia, double tb, int64_t ib) {
    return ta < tb || (ta == tb && ia < ib);
}

#ifndef HP_COARSE
#define HP_COARSE 256
#endif
constexpr int kCoarse = HP_COARSE;


// Block-wide exclusive scan of a[0..n) in place (n <= per * blockDim.x).
template <int kPer>
__device__ void block_scan_inplace(int* a, int n, int* sh) {
    const int tid = threadIdx.x;
    int v[kPer], acc = 0;
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int i = tid * kPer + k;
        v[k] = i < n ? a[i] : 0;
        acc += v[k];
    }
    int total;
    int run = block_excl_scan<int, false>(acc, sh, &total);  // callers sync before sh is reused
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int i = tid * kPer + k;
        if (i < n) a[i] = run;
        run += v[k];
    }
}

// Sort one ray's q matches by (t, id): read from the fill scratch (st, sid,
// sd), write the sorted segment to the outputs.  Buckets are equalised: a
// 256-bin coarse histogram of t over [tmin, tmax] assigns each coarse bin a
// share of the q fine buckets proportional to its population, and t is
// placed linearly inside its bin's share.  The map is monotone in t, so
// buckets are ordered; each element's final position is its bucket start
// plus its exact (t, id) rank among the (few) members of its bucket.
// The (t, id) order of q elements staged in shared memory -> perm[0, q):
// q <= 64 by direct ranks; else an equalised bucket map of t (256-bin coarse
// histogram over the float bounds [tlo, thi] -> q fine buckets allotted in
// proportion -> linear inside a bin; fp32, every step monotone) and an exact
// rank inside each bucket.  hist needs kCap + 1 entries; chist kCoarse + 1
// (both zeroed by the caller when q > 64).  Ends with a barrier.
// kPreCoarse: the caller has already placed every element's coarse
// coordinate in bk[] and counted chist (with coarse_of below), and synced.
__device__ __forceinline__ float coarse_of(double t, float tlo, float cscale) {
    return fminf((__double2float_rn(t) - tlo) * cscale, float(kCoarse));
}
__device__ __forceinline__ float coarse_scale(float tlo, float thi) {
    const float span = thi - tlo;
    // capped so that 0 * scale stays 0 when the span is tiny
    return span > 0.0f ? fminf(float(kCoarse) / span, FLT_MAX) : 0.0f;
}

template <int kCap, int kT, bool kPreCoarse = false>
__device__ void rank_segment(int q, float tlo, float thi, const double* t, const int* id, unsigned* bk, int* hist,
                             unsigned short* lst, unsigned short* perm, int* chist, int* scan_sh) {
    const int tid = threadIdx.x;
    if (q <= 64) {
        for (int e = tid; e < q; e += kT) {
            const double te = t[e];
            const int ie = id[e];
            int rank = 0;
            for (int k = 0; k < q; k++) rank += key_less(t[k], id[k], te, ie);
            perm[rank] = (unsigned short)e;
        }
        __syncthreads();
    } else {
        const int nb = q;  // fine buckets
        // float bounds of the segment's t, from the streaming pass (any
        // monotone bucket map gives the same order: exact in-bucket ranks)
        // The map is computed in fp32 (each step is monotone under round to
        // nearest: float(t), - tlo, * scale, fminf), once per element; the
        // coarse coordinate is kept in bk[] for the fine pass.
        if (!kPreCoarse) {
            const float cscale = coarse_scale(tlo, thi);
            for (int e = tid; e < q; e += kT) {
                const float x = coarse_of(t[e], tlo, cscale);
                bk[e] = __float_as_uint(x);
                const int b = min(int(x), kCoarse - 1);
                const unsigned peers = __match_any_sync(__activemask(), b);
                if (lane_id() == __ffs(peers) - 1) atomicAdd(&chist[b], __popc(peers));
            }
            __syncthreads();
        }
        // coarse prefix counts -> first fine bucket of each coarse bin
        if (tid < 32) {
            int run = 0;
            for (int c0 = 0; c0 < kCoarse; c0 += 32) {
                const int v = chist[c0 + tid];
                const int inc = warp_incl_scan(v);
                chist[c0 + tid] = int((int64_t(run + inc - v) * nb) / q);
                run += __shfl_sync(0xffffffffu, inc, 31);
            }
            if (tid == 0) chist[kCoarse] = nb;
        }
        __syncthreads();
        for (int e = tid; e < q; e += kT) {
            const float x = __uint_as_float(bk[e]);
            const int b = min(int(x), kCoarse - 1);
            const int f0 = chist[b], width = chist[b + 1] - f0;
            int f = f0;
            if (width > 1) {
                // x - b is exact (Sterbenz) and in [0, 1]
                const int off = int((x - float(b)) * float(width));
                f += min(off, width - 1);
            }
            f = min(f, nb - 1);
            HP_ASSERT(f >= 0 && f < nb);
            const int li = atomicAdd(&hist[f], 1);
            bk[e] = (unsigned(f) << 16) | unsigned(li);
        }
        __syncthreads();
        block_scan_inplace<(kCap + kT - 1) / kT>(hist, nb, scan_sh);
        __syncthreads();
        for (int e = tid; e < q; e += kT) {
            const unsigned be_k = bk[e];
            HP_ASSERT(hist[be_k >> 16] + int(be_k & 0xffffu) < q);
            lst[hist[be_k >> 16] + (be_k & 0xffffu)] = (unsigned short)e;
        }
        __syncthreads();
        for (int e = tid; e < q; e += kT) {
            const unsigned be_k = bk[e];
            const int bs = hist[be_k >> 16];
            const int be = (int(be_k >> 16) + 1 < nb) ? hist[(be_k >> 16) + 1] : q;
            int rank = 0;
            if (be - bs > 1) {
                const double te = t[e];
                const int ie = id[e];
                for (int k = bs; k < be; k++) {
                    const int o = lst[k];
                    rank += key_less(t[o], id[o], te, ie);
                }
            }
            HP_ASSERT(bs + rank < q);
            perm[bs + rank] = (unsigned short)e;
        }
        __syncthreads();
    }
}

__device__ __forceinline__ unsigned long long dkey(double x) {  // order-preserving key
    const unsigned long long b = __double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    return __longlong_as_double((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
}


QCam make_qcam(const hp_camera* cam) {
    QCam q{};
    q.has_cam = cam != nullptr;
    if (cam) {
        for (int k = 0; k < 3; k++) {
            q.C.r[k] = cam->right[k];
            q.C.u[k] = cam->up[k];
            q.C.f[k] = cam->forward[k];
        }
        q.C.focal = cam->focal_length;
        q.C.pw = cam->pixel_width;
        q.C.ph = cam->pixel_height;
        q.C.half_w = 0.5 * double(cam->width);
        q.C.half_h = 0.5 * double(cam->height);
        q.width = int(cam->width);
        q.height = int(cam->height);
    }
    return q;
}

int check_common(const hp_query_layout& L, int64_t pad, int64_t m, int64_t wp, int64_t hp) {
    if (pad < 0 || m < 0 || !L.row_ptr || wp < 0 || hp < 0) {
        set_error("hp_query: invalid arguments");
        return HP_EINVAL;
    }
    if (wp * hp >= (int64_t(1) << 31)) {  // row pointers are int32 (hp_build rejects such grids)
        set_error("hp_query: padded grid must be below 2^31 pixels");
        return HP_EINVAL;
    }
    if (2 * pad + 1 > 0xFFFF) {
        set_error("hp_query: kernel too large");
        return HP_EINVAL;
    }
    return HP_OK;
}

unsigned group_grid(int64_t m, int per_sm) {
    const int64_t groups = (m + kGroupMax - 1) / kGroupMax;
    const int64_t cap = int64_t(device_sms()) * per_sm;
    return unsigned(groups < cap ? (groups > 0 ? groups : 1) : cap);
}

// offsets[m] = -(scratch slots needed) when the caller's capacity is short
__global__ void k_mark_overflow(const int64_t* __restrict__ need_at, int64_t capacity, int64_t* __restrict__ total) {
    if (*need_at > capacity) *total = -*need_at;
}

// ---------------------------------------------------------------- pass 0
// Per-ray upper bound of the matches: the number of slots the streaming pass
// will test for the ray (its footprint rows, exactly as stream_group
// tabulates them).  Places each ray's unsorted-match scratch segment.
__global__ void __launch_bounds__(kThreads) k_query_bound(hp_query_layout L, int64_t wp, int pad, Rays R, QCam QC,
                                                          int64_t m, int64_t* __restrict__ bound) {
    __shared__ GroupHead head;
    __shared__ int acc[kGroupMax];
    const int s = 2 * pad + 1;
    for (int64_t r0 = int64_t(blockIdx.x) * kGroupMax; r0 < m; r0 += int64_t(gridDim.x) * kGroupMax) {
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        if (threadIdx.x < kGroupMax) acc[threadIdx.x] = 0;
        group_setup(head, R, QC, r0, G, s);
        for (int idx = threadIdx.x; idx < s * G; idx += kThreads) {
            const int row = idx / G, g = idx - row * G;
            const RayParams& r = head.ray[g];
            const int y = r.v + row;
            int x0, x1;
            if (footprint_row(head.fp[g], QC.C, pad, QC.width, QC.height, r.u, r.v, y, x0, x1)) {
                const int64_t base = int64_t(y) * wp;
                const int n = L.row_ptr[base + x1 + 1] - L.row_ptr[base + x0];
                if (n > 0) atomicAdd(&acc[g], n);
            }
        }
        __syncthreads();
        if (threadIdx.x < G) bound[r0 + threadIdx.x] = acc[threadIdx.x];
        __syncthreads();
    }
}

}  // namespace
}  // namespace hp
