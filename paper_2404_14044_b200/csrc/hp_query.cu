// hp_query.cu — per-ray cone query over the hash index (two passes).
//
// Reference: _kernels.hash_query_batch (_kernels.py:86-157), _cone_test
// (:22-36), _canonical_sort (:39-73).
//
// Data layout (built by hp_build): points re-laid out row-major by padded
// pixel (hp_query_layout), so the s pixels of one kernel row are ONE
// contiguous slot range [row_ptr[y*Wp + u], row_ptr[y*Wp + u + s]).
//
// Work decomposition: a CTA owns a GROUP of consecutive rays (up to 32; for
// ray_grid input these are horizontally adjacent pixels) and streams the
// union of their kernel rows through shared memory, one padded image row at a
// time.  Every staged point is cone-tested by every ray of the group whose
// window covers it (~18 rays for s = 41, G = 32), so L2 traffic is ~1/18 of a
// per-ray scan.
//
//   pass 1 (hp_query_count): exact per-ray match count, probes (= s*s) and
//          scanned (sum of table counts over the window); offsets = scan.
//   pass 2 (hp_query_fill):  rays regrouped so a group's matches fit in
//          shared memory; matches are appended per ray, sorted by (t, id)
//          in shared memory (bucket by t + exact in-bucket rank) and written
//          once, coalesced.  Rays with more matches than fit are handled by
//          a global-memory path (in-place sorting network).
//
// The cone test is fp64 with the reference's operation order and no FMA, so
// ids, t_proj and dist_perp are bit-identical to the reference.
#include <cfloat>
#include <climits>

#include "hp_common.cuh"
#include "hp_sortnet.cuh"

namespace hp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kGroupMax = 32;     // rays per group
constexpr int kStage = 1024;      // staged points per chunk of a row
constexpr int kFillCap = 4096;    // matches buffered per fill group
constexpr int kBucketMax = 2048;  // buckets for the per-ray sort

struct Rays {
    const int64_t* pix;
    int64_t pstride;
    const double* dirs;
    const double* tn;
    const double* tf;
    const double* slopes;
};

struct RayParams {
    int u, v;  // padded window origin (== unpadded pixel)
    double d0, d1, d2, tn, tf, slope;
};

// _cone_test (_kernels.py:22-36): t = p.d; reject outside [tn, tf]; reject
// when |p - t d|^2 > (t * slope)^2.  Returns the exact fp64 t and dist^2.
__device__ __forceinline__ bool cone_test(double p0, double p1, double p2, const RayParams& r,
                                          double& t, double& dist2) {
    t = dadd(dadd(dmul(p0, r.d0), dmul(p1, r.d1)), dmul(p2, r.d2));
    if (t < r.tn || t > r.tf) return false;
    const double e0 = dsub(p0, dmul(t, r.d0));
    const double e1 = dsub(p1, dmul(t, r.d1));
    const double e2 = dsub(p2, dmul(t, r.d2));
    dist2 = dadd(dadd(dmul(e0, e0), dmul(e1, e1)), dmul(e2, e2));
    const double rad = dmul(t, r.slope);
    return !(dist2 > dmul(rad, rad));
}

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
    return p;
}

// Shared state of one streamed group.
struct GroupSmem {
    RayParams ray[kGroupMax];
    int lo[kGroupMax], hi[kGroupMax];  // the ray's slot sub-range in the current row
    double px[kStage], py[kStage], pz[kStage];
    int pid[kStage];
    int stage_lo, stage_hi, u0, u1, v0, v1;
};

// Streams the rows of a group; calls visit(ray_slot, slot_index_in_stage, t,
// dist2) for every accepted (ray, point) pair, on the warp that owns the ray
// (warp w owns rays w, w+8, ...).  `with_ids` stages point ids as well.
template <bool kWithIds, class Visit, class RowDone>
__device__ void stream_group(GroupSmem& S, int G, const hp_query_layout L, int64_t wp, int s,
                             Visit visit, RowDone row_done) {
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    for (int y = S.v0; y < S.v1; y++) {
        const int64_t rowbase = int64_t(y) * wp;
        // each ray's sub-range of this row (rays outside the row: empty)
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
            S.stage_lo = L.row_ptr[rowbase + S.u0];
            S.stage_hi = L.row_ptr[rowbase + S.u1];
        }
        __syncthreads();
        const int A = S.stage_lo, B = S.stage_hi;
        for (int c0 = A; c0 < B; c0 += kStage) {
            const int c1 = c0 + kStage < B ? c0 + kStage : B;
            for (int k = c0 + tid; k < c1; k += kThreads) {
                S.px[k - c0] = L.rel_x[k];
                S.py[k - c0] = L.rel_y[k];
                S.pz[k - c0] = L.rel_z[k];
                if (kWithIds) S.pid[k - c0] = L.point_id[k];
            }
            __syncthreads();
            for (int g = warp; g < G; g += kWarps) {
                const int lo = max(S.lo[g], c0), hi = min(S.hi[g], c1);
                if (lo >= hi) continue;
                const RayParams r = S.ray[g];
                for (int base = lo; base < hi; base += 32) {
                    const int k = base + lane;
                    double t = 0.0, d2 = 0.0;
                    bool ok = false;
                    if (k < hi) ok = cone_test(S.px[k - c0], S.py[k - c0], S.pz[k - c0], r, t, d2);
                    visit(g, k - c0, ok, t, d2);
                }
            }
            __syncthreads();
        }
        row_done(y);
    }
}

// Group bounding box (padded coordinates) of rays [r0, r0+G).
__device__ void group_setup(GroupSmem& S, const Rays& R, int64_t r0, int G, int s) {
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

// ---------------------------------------------------------------- pass 1
__global__ void __launch_bounds__(kThreads) k_query_count(hp_query_layout L, int64_t wp, int pad, Rays R,
                                                          int64_t m, int64_t* __restrict__ counts,
                                                          int64_t* __restrict__ probes,
                                                          int64_t* __restrict__ scanned) {
    __shared__ GroupSmem S;
    __shared__ int64_t cnt[kGroupMax], scn[kGroupMax];
    const int s = 2 * pad + 1;
    for (int64_t r0 = int64_t(blockIdx.x) * kGroupMax; r0 < m; r0 += int64_t(gridDim.x) * kGroupMax) {
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        if (threadIdx.x < kGroupMax) cnt[threadIdx.x] = scn[threadIdx.x] = 0;
        group_setup(S, R, r0, G, s);
        stream_group<false>(
            S, G, L, wp, s,
            [&](int g, int, bool ok, double, double) {
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                if (lane_id() == 0) cnt[g] += __popc(b);
            },
            [&](int) {
                if (threadIdx.x < G) scn[threadIdx.x] += S.hi[threadIdx.x] - S.lo[threadIdx.x];
            });
        __syncthreads();
        if (threadIdx.x < G) {
            counts[r0 + threadIdx.x] = cnt[threadIdx.x];
            probes[r0 + threadIdx.x] = int64_t(s) * s;
            scanned[r0 + threadIdx.x] = scn[threadIdx.x];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- grouping
// Greedy split of every 32-ray chunk into fill groups whose total match count
// fits kFillCap; rays above kFillCap become single "big" groups; groups with
// no matches are dropped.  Descriptor: x = first ray, y = ray count | big<<8.
__global__ void k_make_groups(const int64_t* __restrict__ off, int64_t m, int2* __restrict__ groups,
                              int* __restrict__ ngroups) {
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
    for (int64_t c = blockIdx.x * int64_t(blockDim.x / 32) + warp_id(); c * 32 < m; c += warps) {
        if (lane_id() == 0) {
            int64_t first = c * 32, sum = 0;
            int n = 0;
            const int len = int(m - c * 32 < 32 ? m - c * 32 : 32);
            for (int k = 0; k < len; k++) {
                const int64_t qk = off[c * 32 + k + 1] - off[c * 32 + k];
                if (qk > kFillCap) {
                    if (n && sum) groups[atomicAdd(ngroups, 1)] = make_int2(int(first), n);
                    groups[atomicAdd(ngroups, 1)] = make_int2(int(c * 32 + k), 1 | (1 << 8));
                    first = c * 32 + k + 1;
                    n = 0;
                    sum = 0;
                    continue;
                }
                if (sum + qk > kFillCap) {
                    if (sum) groups[atomicAdd(ngroups, 1)] = make_int2(int(first), n);
                    first = c * 32 + k;
                    n = 0;
                    sum = 0;
                }
                sum += qk;
                n++;
            }
            if (n && sum) groups[atomicAdd(ngroups, 1)] = make_int2(int(first), n);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- pass 2
struct FillSmem {
    double t[kFillCap];
    double d[kFillCap];
    int id[kFillCap];
    unsigned short lst[kFillCap];
    unsigned short perm[kFillCap];
    unsigned int bk[kFillCap];  // bucket << 16 | local index
    int hist[kBucketMax + 1];
    int base[kGroupMax + 1];  // region of each ray in the buffers
    int fill[kGroupMax];
    int64_t out_off[kGroupMax];
    unsigned long long tmin, tmax;
    int scan_sh[kWarps + 1];
};

__device__ __forceinline__ bool key_less(double ta, int ia, double tb, int ib) {
    return ta < tb || (ta == tb && ia < ib);
}

// Sort the q matches of one ray (region [b0, b0+q) of the buffers) by
// (t, id) and write them to the output segment at `off`.  Block-wide.
__device__ void sort_and_write(FillSmem& F, int b0, int q, int64_t off, int64_t* __restrict__ out_id,
                               double* __restrict__ out_t, double* __restrict__ out_d) {
    const int tid = threadIdx.x;
    if (q <= 64) {
        // direct rank: each element counts the elements ordered before it
        for (int e = tid; e < q; e += kThreads) {
            const double te = F.t[b0 + e];
            const int ie = F.id[b0 + e];
            int rank = 0;
            for (int k = 0; k < q; k++) rank += key_less(F.t[b0 + k], F.id[b0 + k], te, ie);
            F.perm[b0 + rank] = (unsigned short)e;
        }
        __syncthreads();
    } else {
        int nb = 64;
        while (nb < q && nb < kBucketMax) nb <<= 1;
        if (tid == 0) {
            F.tmin = ~0ull;
            F.tmax = 0ull;
        }
        for (int k = tid; k <= nb; k += kThreads) F.hist[k] = 0;
        __syncthreads();
        unsigned long long lmin = ~0ull, lmax = 0;
        for (int e = tid; e < q; e += kThreads) {
            const unsigned long long kk = okey(F.t[b0 + e]);
            lmin = lmin < kk ? lmin : kk;
            lmax = lmax > kk ? lmax : kk;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            unsigned long long a = __shfl_xor_sync(0xffffffffu, lmin, o), b = __shfl_xor_sync(0xffffffffu, lmax, o);
            lmin = lmin < a ? lmin : a;
            lmax = lmax > b ? lmax : b;
        }
        if (lane_id() == 0) {
            atomicMin(&F.tmin, lmin);
            atomicMax(&F.tmax, lmax);
        }
        __syncthreads();
        // okey is invertible: recover the doubles
        const unsigned long long kmin = F.tmin, kmax = F.tmax;
        const double tlo = __longlong_as_double((kmin & 0x8000000000000000ull) ? (kmin & 0x7fffffffffffffffull) : ~kmin);
        const double thi = __longlong_as_double((kmax & 0x8000000000000000ull) ? (kmax & 0x7fffffffffffffffull) : ~kmax);
        const double span = dsub(thi, tlo);
        // capped so that 0 * scale stays 0 when the span is tiny
        const double scale = span > 0.0 ? fmin(__ddiv_rn(double(nb), span), DBL_MAX) : 0.0;
        for (int e = tid; e < q; e += kThreads) {
            // monotone in t: (t - tlo) and the positive scaling both preserve order
            const double x = fmin(dmul(dsub(F.t[b0 + e], tlo), scale), double(nb - 1));
            const int b = int(x);
            const int li = atomicAdd(&F.hist[b], 1);
            F.bk[b0 + e] = (unsigned(b) << 16) | unsigned(li);
        }
        __syncthreads();
        // exclusive scan of hist[0..nb) (nb <= kBucketMax = 8 per thread)
        {
            constexpr int kPer = kBucketMax / kThreads;
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
            const unsigned bk = F.bk[b0 + e];
            F.lst[b0 + F.hist[bk >> 16] + (bk & 0xffffu)] = (unsigned short)e;
        }
        __syncthreads();
        for (int e = tid; e < q; e += kThreads) {
            const unsigned bk = F.bk[b0 + e];
            const int bs = F.hist[bk >> 16];
            const int be = (int(bk >> 16) + 1 < nb) ? F.hist[(bk >> 16) + 1] : q;
            const double te = F.t[b0 + e];
            const int ie = F.id[b0 + e];
            int rank = 0;
            for (int k = bs; k < be; k++) {
                const int o = F.lst[b0 + k];
                rank += key_less(F.t[b0 + o], F.id[b0 + o], te, ie);
            }
            F.perm[b0 + bs + rank] = (unsigned short)e;
        }
        __syncthreads();
    }
    for (int p = tid; p < q; p += kThreads) {
        const int e = F.perm[b0 + p];
        out_id[off + p] = F.id[b0 + e];
        out_t[off + p] = F.t[b0 + e];
        out_d[off + p] = F.d[b0 + e];
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_query_fill(hp_query_layout L, int64_t wp, int pad, Rays R,
                                                         const int64_t* __restrict__ off,
                                                         const int2* __restrict__ groups,
                                                         const int* __restrict__ ngroups,
                                                         int* __restrict__ work, int64_t* __restrict__ out_id,
                                                         double* __restrict__ out_t, double* __restrict__ out_d) {
    __shared__ GroupSmem S;
    extern __shared__ __align__(16) unsigned char dyn[];
    FillSmem& F = *reinterpret_cast<FillSmem*>(dyn);
    __shared__ int gidx;
    const int s = 2 * pad + 1;
    const int ng = *ngroups;
    for (;;) {
        if (threadIdx.x == 0) gidx = atomicAdd(work, 1);
        __syncthreads();
        const int gi = gidx;
        __syncthreads();
        if (gi >= ng) break;
        const int2 gd = groups[gi];
        const int64_t r0 = gd.x;
        const int G = gd.y & 0xff;
        const bool big = (gd.y >> 8) & 1;
        group_setup(S, R, r0, G, s);
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int g = 0; g < G; g++) {
                F.base[g] = acc;
                F.fill[g] = 0;
                F.out_off[g] = off[r0 + g];
                acc += int(off[r0 + g + 1] - off[r0 + g]);
            }
            F.base[G] = acc;
        }
        __syncthreads();
        if (!big) {
            stream_group<true>(
                S, G, L, wp, s,
                [&](int g, int k, bool ok, double t, double d2) {
                    const unsigned b = __ballot_sync(0xffffffffu, ok);
                    if (ok) {
                        const int pos = F.base[g] + F.fill[g] + __popc(b & ((1u << lane_id()) - 1));
                        F.t[pos] = t;
                        F.d[pos] = sqrt(d2);
                        F.id[pos] = S.pid[k];
                    }
                    __syncwarp();
                    if (lane_id() == 0) F.fill[g] += __popc(b);
                    __syncwarp();
                },
                [&](int) {});
            __syncthreads();
            for (int g = 0; g < G; g++) {
                const int q = F.base[g + 1] - F.base[g];
                if (q == 0) continue;
                sort_and_write(F, F.base[g], q, F.out_off[g], out_id, out_t, out_d);
            }
        } else {
            // one ray with more matches than the shared buffer: append into the
            // output segment (unsorted), then sort it in place in global memory.
            const int64_t o = F.out_off[0];
            stream_group<true>(
                S, 1, L, wp, s,
                [&](int, int k, bool ok, double t, double d2) {
                    const unsigned b = __ballot_sync(0xffffffffu, ok);
                    if (ok) {
                        const int64_t pos = o + F.fill[0] + __popc(b & ((1u << lane_id()) - 1));
                        out_t[pos] = t;
                        out_d[pos] = sqrt(d2);
                        out_id[pos] = S.pid[k];
                    }
                    __syncwarp();
                    if (lane_id() == 0) F.fill[0] += __popc(b);
                    __syncwarp();
                },
                [&](int) {});
            __syncthreads();
            const int64_t q = off[r0 + 1] - off[r0];
            double* tt = out_t + o;
            double* dd = out_d + o;
            int64_t* ii = out_id + o;
            block_bitonic_sort(
                q, [&](int64_t a, int64_t b) { return tt[a] < tt[b] || (tt[a] == tt[b] && ii[a] < ii[b]); },
                [&](int64_t a, int64_t b) {
                    double x = tt[a]; tt[a] = tt[b]; tt[b] = x;
                    x = dd[a]; dd[a] = dd[b]; dd[b] = x;
                    int64_t y = ii[a]; ii[a] = ii[b]; ii[b] = y;
                });
        }
        __syncthreads();
    }
}

struct QueryWs {
    int2* groups;
    int* ngroups;
    int* work;
    void* scan;
};

QueryWs carve_query(Carver& c, int64_t m) {
    QueryWs w;
    w.groups = c.take<int2>(m > 0 ? m : 1);
    w.ngroups = c.take<int>(1);
    w.work = c.take<int>(1);
    w.scan = c.take<char>(scan_workspace_bytes(m + 1));
    return w;
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

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_query_workspace_bytes(int64_t m, int64_t pad, size_t* bytes) {
    Carver c(nullptr, 0);
    carve_query(c, m);
    *bytes = c.used + 256;
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
    Carver c(workspace, workspace_bytes);
    QueryWs w = carve_query(c, m);
    if (!c.ok()) {
        set_error("hp_query_count: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    if (m > 0) {
        const int64_t groups = (m + kGroupMax - 1) / kGroupMax;
        const unsigned grid = unsigned(groups < 148 * 8 ? groups : 148 * 8);
        k_query_count<<<grid, kThreads, 0, s>>>(layout, padded_w, int(pad), R, m, offsets, probes, scanned);
        HP_CHECK_LAUNCH("k_query_count");
    }
    HP_TRY(exclusive_scan_i64(offsets, offsets, m, w.scan, s));
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
    if (m == 0 || total == 0) return HP_OK;
    Carver c(workspace, workspace_bytes);
    QueryWs w = carve_query(c, m);
    if (!c.ok()) {
        set_error("hp_query_fill: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    if (cudaMemsetAsync(w.ngroups, 0, sizeof(int), s) != cudaSuccess ||
        cudaMemsetAsync(w.work, 0, sizeof(int), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_query_fill memset");
    const int64_t chunks = (m + 31) / 32;
    k_make_groups<<<grid_for(chunks * 32, 256), 256, 0, s>>>(offsets, m, w.groups, w.ngroups);
    HP_CHECK_LAUNCH("k_make_groups");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_query_fill, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(FillSmem)));
        attr = true;
    }
    k_query_fill<<<148 * 2, kThreads, sizeof(FillSmem), s>>>(layout, padded_w, int(pad), R, offsets, w.groups,
                                                              w.ngroups, w.work, ids, t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_fill");
    return HP_OK;
}
