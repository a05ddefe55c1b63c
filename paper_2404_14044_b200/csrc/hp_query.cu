// hp_query.cu — per-ray cone query over the hash index.
//
// Reference: _kernels.hash_query_batch (_kernels.py:86-157), _cone_test
// (:22-36), _canonical_sort (:39-73).
//
// Data layout (built by hp_build): points re-laid out row-major by padded
// pixel (hp_query_layout), so the s pixels of one kernel row are ONE
// contiguous slot range [row_ptr[y*Wp + u], row_ptr[y*Wp + u + s]).
//
// Work decomposition: a CTA owns a GROUP of up to 32 consecutive rays (for
// ray_grid input: horizontally adjacent pixels) and streams the union of
// their kernel rows through shared memory, one padded image row at a time.
// Every staged point is tested by every ray of the group whose window covers
// it (~18 rays for s = 41), so L2 traffic is ~1/18 of a per-ray scan.
//
// Cone test: a float32 filter with a rigorous error budget classifies each
// (ray, point) pair as sure-reject / sure-accept / uncertain (DESIGN.md "fp32
// filter"); the reference's fp64 test (same operation order, no FMA) decides
// the uncertain pairs and produces the exact t_proj / dist_perp of accepted
// ones, so results are bit-identical to the reference.
//
//   k_query_count  exact per-ray count, probes (= s*s), scanned; offsets = scan
//   k_query_fill   same streaming; accepted pairs written (unsorted) into the
//                  ray's CSR segment
//   k_query_sort   per ray: (t, id) sort of its segment in shared memory
//                  (bucket by t + exact in-bucket rank), in place; segments
//                  longer than the shared buffer use an in-place sorting
//                  network in global memory
#include <math_constants.h>

#include <cfloat>
#include <climits>

#include "hp_common.cuh"
#include "hp_cone.cuh"
#include "hp_sortnet.cuh"

namespace hp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroupMax = 32;  // rays per group
constexpr int kStageCount = 2048;
constexpr int kStageFill = 512;

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

struct GroupHead {
    RayParams ray[kGroupMax];
    int lo[kGroupMax], hi[kGroupMax];  // the ray's slot sub-range in the current row
    int stage_lo[2], stage_hi[2];  // by row parity (no end-of-row barrier needed)
    int u0, u1, v0, v1;
};

// Group bounding box (padded coordinates) of rays [r0, r0+G).
__device__ void group_setup(GroupHead& S, const Rays& R, int64_t r0, int G, int s) {
    const int tid = threadIdx.x;
    if (tid < G) S.ray[tid] = load_ray(R, r0 + tid);
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

// Streams the kernel rows of a group.  For each staged chunk of a row,
// stage(c0, c1) loads slots [c0, c1) into shared memory, then every warp
// calls test(g, k, c0) for the rays g it owns (warp w owns rays w, w+8, ...)
// over their sub-range, 32 slots at a time (lanes beyond the range get
// k = -1).  row_done() runs once per row after the ranges are known.
template <int kStage, class Stage, class Test, class RowDone>
__device__ void stream_group(GroupHead& S, int G, const hp_query_layout L, int64_t wp, int s, Stage stage,
                             Test test, RowDone row_done) {
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    for (int y = S.v0; y < S.v1; y++) {
        const int64_t rowbase = int64_t(y) * wp;
        if (tid < G) {
            const RayParams& r = S.ray[tid];
            if (y >= r.v && y < r.v + s) {
                S.lo[tid] = L.row_ptr[rowbase + r.u];
                S.hi[tid] = L.row_ptr[rowbase + r.u + s];
            } else {
                S.lo[tid] = S.hi[tid] = 0;
            }
        }
        if (tid == 0) {
            S.stage_lo[y & 1] = L.row_ptr[rowbase + S.u0];
            S.stage_hi[y & 1] = L.row_ptr[rowbase + S.u1];
        }
        __syncthreads();
        row_done();
        const int A = S.stage_lo[y & 1], B = S.stage_hi[y & 1];
        for (int c0 = A; c0 < B; c0 += kStage) {
            const int c1 = c0 + kStage < B ? c0 + kStage : B;
            stage(c0, c1);
            __syncthreads();
            for (int g = warp; g < G; g += kWarps) {
                const int lo = max(S.lo[g], c0), hi = min(S.hi[g], c1);
                for (int base = lo; base < hi; base += 32) {
                    const int k = base + lane;
                    test(g, k < hi ? k : -1, c0);
                }
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- pass 1
struct CountSmem {
    GroupHead head;
    float4 pf[kStageCount];
    int64_t cnt[kGroupMax], scn[kGroupMax];
};

__global__ void __launch_bounds__(kThreads) k_query_count(hp_query_layout L, int64_t wp, int pad, Rays R,
                                                          int64_t m, int64_t* __restrict__ counts,
                                                          int64_t* __restrict__ probes,
                                                          int64_t* __restrict__ scanned) {
    extern __shared__ __align__(16) unsigned char dyn[];
    CountSmem& S = *reinterpret_cast<CountSmem*>(dyn);
    const int s = 2 * pad + 1;
    const float4* __restrict__ relf = reinterpret_cast<const float4*>(L.relf);
    for (int64_t r0 = int64_t(blockIdx.x) * kGroupMax; r0 < m; r0 += int64_t(gridDim.x) * kGroupMax) {
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        if (threadIdx.x < kGroupMax) S.cnt[threadIdx.x] = S.scn[threadIdx.x] = 0;
        group_setup(S.head, R, r0, G, s);
        stream_group<kStageCount>(
            S.head, G, L, wp, s,
            [&](int c0, int c1) {
                for (int k = c0 + int(threadIdx.x); k < c1; k += kThreads) S.pf[k - c0] = relf[k];
            },
            [&](int g, int k, int c0) {
                int cls = 0;
                if (k >= 0) {
                    const RayParams& r = S.head.ray[g];
                    cls = cone_filter(S.pf[k - c0], r);
                    if (cls == 2) {
                        double t, d2;
                        cls = cone_test(L.rel_x[k], L.rel_y[k], L.rel_z[k], r, t, d2) ? 1 : 0;
                    }
                }
                const unsigned b = __ballot_sync(0xffffffffu, cls == 1);
                if (lane_id() == 0) S.cnt[g] += __popc(b);
            },
            [&]() {
                if (threadIdx.x < G) S.scn[threadIdx.x] += S.head.hi[threadIdx.x] - S.head.lo[threadIdx.x];
            });
        __syncthreads();
        if (threadIdx.x < G) {
            counts[r0 + threadIdx.x] = S.cnt[threadIdx.x];
            probes[r0 + threadIdx.x] = int64_t(s) * s;
            scanned[r0 + threadIdx.x] = S.scn[threadIdx.x];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- pass 2
struct FillSmem {
    GroupHead head;
    float4 pf[kStageFill];
    double px[kStageFill], py[kStageFill], pz[kStageFill];
    int pid[kStageFill];
    int fill[kGroupMax];
    int64_t off[kGroupMax];
};

__global__ void __launch_bounds__(kThreads) k_query_fill(hp_query_layout L, int64_t wp, int pad, Rays R,
                                                         int64_t m, const int64_t* __restrict__ off,
                                                         int64_t* __restrict__ out_id, double* __restrict__ out_t,
                                                         double* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char dyn[];
    FillSmem& S = *reinterpret_cast<FillSmem*>(dyn);
    const int s = 2 * pad + 1;
    const float4* __restrict__ relf = reinterpret_cast<const float4*>(L.relf);
    for (int64_t r0 = int64_t(blockIdx.x) * kGroupMax; r0 < m; r0 += int64_t(gridDim.x) * kGroupMax) {
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        // skip groups without matches
        const int64_t total = off[r0 + G] - off[r0];
        if (total == 0) continue;
        if (threadIdx.x < G) {
            S.fill[threadIdx.x] = 0;
            S.off[threadIdx.x] = off[r0 + threadIdx.x];
        }
        group_setup(S.head, R, r0, G, s);
        stream_group<kStageFill>(
            S.head, G, L, wp, s,
            [&](int c0, int c1) {
                for (int k = c0 + int(threadIdx.x); k < c1; k += kThreads) {
                    S.pf[k - c0] = relf[k];
                    S.px[k - c0] = L.rel_x[k];
                    S.py[k - c0] = L.rel_y[k];
                    S.pz[k - c0] = L.rel_z[k];
                    S.pid[k - c0] = L.point_id[k];
                }
            },
            [&](int g, int k, int c0) {
                int cls = 0;
                double t = 0.0, d2 = 0.0;
                if (k >= 0) {
                    const RayParams& r = S.head.ray[g];
                    const int i = k - c0;
                    cls = cone_filter(S.pf[i], r);
                    if (cls != 0) {
                        const bool ok = cone_test(S.px[i], S.py[i], S.pz[i], r, t, d2);
                        if (cls == 2) cls = ok ? 1 : 0;
                    }
                }
                const unsigned b = __ballot_sync(0xffffffffu, cls == 1);
                if (cls == 1) {
                    const int64_t pos = S.off[g] + S.fill[g] + __popc(b & ((1u << lane_id()) - 1));
                    out_t[pos] = t;
                    out_d[pos] = sqrt(d2);
                    out_id[pos] = S.pid[k - c0];
                }
                __syncwarp();
                if (lane_id() == 0) S.fill[g] += __popc(b);
                __syncwarp();
            },
            [&]() {});
        __syncthreads();
    }
}

// ---------------------------------------------------------------- sort
__device__ __forceinline__ bool key_less(double ta, int64_t ia, double tb, int64_t ib) {
    return ta < tb || (ta == tb && ia < ib);
}

template <int kCap>
struct SortSmem {
    double t[kCap];
    int id[kCap];  // point ids < 2^31 (hp_build)
    unsigned int bk[kCap];  // bucket << 16 | local index
    unsigned short lst[kCap];
    unsigned short perm[kCap];
    int hist[kCap + 1];
    unsigned long long tmin, tmax;
    int scan_sh[kWarps + 1];
};

// Sort one ray's segment [off, off+q) by (t, id) in place (q <= kCap).
template <int kCap>
__device__ void sort_segment(SortSmem<kCap>& F, int q, int64_t* __restrict__ gid, double* __restrict__ gt,
                             double* __restrict__ gd) {
    constexpr int kPer = (kCap + kThreads - 1) / kThreads;
    const int tid = threadIdx.x;
    for (int e = tid; e < q; e += kThreads) {
        F.t[e] = gt[e];
        F.id[e] = int(gid[e]);
    }
    if (q <= 64) {
        __syncthreads();
        for (int e = tid; e < q; e += kThreads) {
            const double te = F.t[e];
            const int ie = F.id[e];
            int rank = 0;
            for (int k = 0; k < q; k++) rank += key_less(F.t[k], F.id[k], te, ie);
            F.perm[rank] = (unsigned short)e;
        }
        __syncthreads();
    } else {
        int nb = 64;
        while (nb < q && nb < kCap) nb <<= 1;
        if (tid == 0) {
            F.tmin = ~0ull;
            F.tmax = 0ull;
        }
        for (int k = tid; k <= nb; k += kThreads) F.hist[k] = 0;
        __syncthreads();
        unsigned long long lmin = ~0ull, lmax = 0;
        for (int e = tid; e < q; e += kThreads) {
            const unsigned long long kk = okey(F.t[e]);
            lmin = lmin < kk ? lmin : kk;
            lmax = lmax > kk ? lmax : kk;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xffffffffu, lmin, o);
            const unsigned long long b = __shfl_xor_sync(0xffffffffu, lmax, o);
            lmin = lmin < a ? lmin : a;
            lmax = lmax > b ? lmax : b;
        }
        if (lane_id() == 0) {
            atomicMin(&F.tmin, lmin);
            atomicMax(&F.tmax, lmax);
        }
        __syncthreads();
        const unsigned long long kmin = F.tmin, kmax = F.tmax;
        const double tlo = __longlong_as_double((kmin & 0x8000000000000000ull) ? (kmin & 0x7fffffffffffffffull) : ~kmin);
        const double thi = __longlong_as_double((kmax & 0x8000000000000000ull) ? (kmax & 0x7fffffffffffffffull) : ~kmax);
        const double span = dsub(thi, tlo);
        // capped so that 0 * scale stays 0 when the span is tiny
        const double scale = span > 0.0 ? fmin(__ddiv_rn(double(nb), span), DBL_MAX) : 0.0;
        for (int e = tid; e < q; e += kThreads) {
            // monotone in t: (t - tlo) and the positive scaling both preserve order
            const double x = fmin(dmul(dsub(F.t[e], tlo), scale), double(nb - 1));
            const int b = int(x);
            const int li = atomicAdd(&F.hist[b], 1);
            F.bk[e] = (unsigned(b) << 16) | unsigned(li);
        }
        __syncthreads();
        {
            int v[kPer], acc = 0;
#pragma unroll
            for (int k = 0; k < kPer; k++) {
                const int i = tid * kPer + k;
                v[k] = i < nb ? F.hist[i] : 0;
                acc += v[k];
            }
            int total;
            int run = block_excl_scan<int>(acc, F.scan_sh, &total);
#pragma unroll
            for (int k = 0; k < kPer; k++) {
                const int i = tid * kPer + k;
                if (i < nb) F.hist[i] = run;
                run += v[k];
            }
        }
        __syncthreads();
        for (int e = tid; e < q; e += kThreads) {
            const unsigned bk = F.bk[e];
            F.lst[F.hist[bk >> 16] + (bk & 0xffffu)] = (unsigned short)e;
        }
        __syncthreads();
        for (int e = tid; e < q; e += kThreads) {
            const unsigned bk = F.bk[e];
            const int bs = F.hist[bk >> 16];
            const int be = (int(bk >> 16) + 1 < nb) ? F.hist[(bk >> 16) + 1] : q;
            const double te = F.t[e];
            const int ie = F.id[e];
            int rank = 0;
            for (int k = bs; k < be; k++) {
                const int o = F.lst[k];
                rank += key_less(F.t[o], F.id[o], te, ie);
            }
            F.perm[bs + rank] = (unsigned short)e;
        }
        __syncthreads();
    }
    // dist: gather in permuted order into registers before overwriting
    double dv[kPer];
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int p = tid + k * kThreads;
        if (p < q) dv[k] = gd[F.perm[p]];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; k++) {
        const int p = tid + k * kThreads;
        if (p < q) {
            const int e = F.perm[p];
            gd[p] = dv[k];
            gt[p] = F.t[e];
            gid[p] = F.id[e];
        }
    }
    __syncthreads();
}

// Rays with lo_q < q <= kCap (kCap > 0), or q > lo_q with the in-place global
// network (kCap == 0).
template <int kCap>
__global__ void __launch_bounds__(kThreads) k_query_sort(const int64_t* __restrict__ off, int64_t m, int lo_q,
                                                         int64_t* __restrict__ out_id, double* __restrict__ out_t,
                                                         double* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char dyn[];
    for (int64_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int64_t o = off[r];
        const int64_t q = off[r + 1] - o;
        if (q <= lo_q || q < 2) continue;
        if constexpr (kCap > 0) {
            if (q > kCap) continue;
            sort_segment<kCap>(*reinterpret_cast<SortSmem<kCap>*>(dyn), int(q), out_id + o, out_t + o, out_d + o);
        } else {
            double* tt = out_t + o;
            double* dd = out_d + o;
            int64_t* ii = out_id + o;
            block_bitonic_sort(
                q, [&](int64_t a, int64_t b) { return key_less(tt[a], ii[a], tt[b], ii[b]); },
                [&](int64_t a, int64_t b) {
                    double x = tt[a];
                    tt[a] = tt[b];
                    tt[b] = x;
                    x = dd[a];
                    dd[a] = dd[b];
                    dd[b] = x;
                    const int64_t y = ii[a];
                    ii[a] = ii[b];
                    ii[b] = y;
                });
            __syncthreads();
        }
    }
}

constexpr int kSortSmall = 2048;
constexpr int kSortLarge = 8192;

template <class K>
int set_smem(K kernel, size_t bytes) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    return e == cudaSuccess ? HP_OK : cuda_status(e, "cudaFuncSetAttribute");
}

int check_common(const hp_query_layout& L, int64_t pad, int64_t m) {
    if (pad < 0 || m < 0 || !L.row_ptr) {
        set_error("hp_query: invalid arguments");
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
    const int64_t cap = int64_t(kNumSMs) * per_sm;
    return unsigned(groups < cap ? (groups > 0 ? groups : 1) : cap);
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_query_workspace_bytes(int64_t m, int64_t pad, size_t* bytes) {
    *bytes = scan_workspace_bytes(m + 1) + 256;
    (void)pad;
    return HP_OK;
}

extern "C" int hp_query_count(hp_query_layout layout, int64_t padded_w, int64_t padded_h, int64_t pad,
                              const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                              const double* t_near, const double* t_far, const double* slopes, int64_t m,
                              int64_t* offsets, int64_t* probes, int64_t* scanned, void* workspace,
                              size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(check_common(layout, pad, m));
    (void)padded_h;
    if (workspace_bytes < scan_workspace_bytes(m + 1)) {
        set_error("hp_query_count: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    if (m > 0) {
        static bool attr = false;
        if (!attr) {
            HP_TRY(set_smem(k_query_count, sizeof(CountSmem)));
            attr = true;
        }
        k_query_count<<<group_grid(m, 6), kThreads, sizeof(CountSmem), s>>>(layout, padded_w, int(pad), R, m,
                                                                            offsets, probes, scanned);
        HP_CHECK_LAUNCH("k_query_count");
    }
    HP_TRY(exclusive_scan_i64(offsets, offsets, m, workspace, s));
    return HP_OK;
}

extern "C" int hp_query_fill(hp_query_layout layout, int64_t padded_w, int64_t padded_h, int64_t pad,
                             const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                             const double* t_near, const double* t_far, const double* slopes, int64_t m,
                             const int64_t* offsets, int64_t total, int64_t* ids, double* t_proj,
                             double* dist_perp, void* workspace, size_t workspace_bytes,
                             hp_stream_t stream) {
    HP_TRY(check_common(layout, pad, m));
    (void)padded_h;
    (void)workspace;
    (void)workspace_bytes;
    if (m == 0 || total == 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    static bool attr = false;
    if (!attr) {
        HP_TRY(set_smem(k_query_fill, sizeof(FillSmem)));
        HP_TRY(set_smem(k_query_sort<kSortSmall>, sizeof(SortSmem<kSortSmall>)));
        HP_TRY(set_smem(k_query_sort<kSortLarge>, sizeof(SortSmem<kSortLarge>)));
        attr = true;
    }
    k_query_fill<<<group_grid(m, 4), kThreads, sizeof(FillSmem), s>>>(layout, padded_w, int(pad), R, m, offsets,
                                                                      ids, t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_fill");
    const unsigned g = unsigned(m < int64_t(kNumSMs) * 8 ? m : int64_t(kNumSMs) * 8);
    k_query_sort<kSortSmall><<<g, kThreads, sizeof(SortSmem<kSortSmall>), s>>>(offsets, m, 0, ids, t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_sort<small>");
    k_query_sort<kSortLarge><<<kNumSMs, kThreads, sizeof(SortSmem<kSortLarge>), s>>>(offsets, m, kSortSmall, ids,
                                                                                     t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_sort<large>");
    k_query_sort<0><<<kNumSMs, kThreads, 0, s>>>(offsets, m, kSortLarge, ids, t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_sort<global>");
    return HP_OK;
}
