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
//   k_query_bound  per-ray upper bound of the matches (footprint slots):
//                  scanned into the rays' scratch offsets
//   k_query_scan   the one streaming pass: accepted pairs (t, id, dist) are
//                  appended unsorted to the ray's scratch segment; exact
//                  counts (-> CSR offsets), probes, scanned, float t bounds
//   k_query_sort   per ray (size classes): (t, id) sort of its segment in
//                  shared memory (equalised buckets of t + exact in-bucket
//                  rank) into the CSR; rays above the largest class are
//                  split into t-ordered parts first (k_query_split)
// (hp_query_count = bound + scan, hp_query_fill = sort)
#include <math_constants.h>

#include <cfloat>
#include <climits>

#include "hp_common.cuh"
#include "hp_cone.cuh"
#include "hp_query_core.cuh"
#include "hp_sortnet.cuh"

namespace hp {
namespace {

#ifndef HP_STAGE_FILL
#define HP_STAGE_FILL 384
#endif
#ifndef HP_SCAN_MINB
#define HP_SCAN_MINB 0
#endif
constexpr int kStageFill = HP_STAGE_FILL;


// Streams the kernel rows of a group through two shared-memory stages.
// Rows are processed in batches of kRowsMax: the batch's per-(row, ray) slot
// sub-ranges are tabulated first (one parallel round of row_ptr loads, each
// ray's total added to `scanned` via tab(g, hi - lo)), then the batch's
// chunks (row, [c0, c1)) are staged with cp.async into alternating buffers:
// chunk i+1 is in flight while chunk i is tested.  issue(buf, c0, c1) issues
// the copies of slots [c0, c1); test(buf, g, lo, hi, c0) runs on the warp
// owning ray g (warp w owns rays w, w+8, ...) over the ray's non-empty slot
// sub-range [lo, hi) of the chunk staged at c0.
template <int kStage, class Issue, class Test, class Tab, class Done>
__device__ void stream_group(GroupHead& S, int G, const hp_query_layout L, int64_t wp, int s, const QCam& QC,
                             Issue issue, Test test, Tab tab, Done done) {
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    const int pad = (s - 1) / 2;
    for (int yb = S.v0; yb < S.v1; yb += kRowsMax) {
        const int nrows = min(kRowsMax, S.v1 - yb);
        for (int row = tid; row < nrows; row += kThreads) {
            S.slo[row] = INT_MAX;
            S.shi[row] = INT_MIN;
        }
        __syncthreads();
        for (int idx = tid; idx < nrows * G; idx += kThreads) {
            const int row = idx / G, g = idx - row * G;
            const int y = yb + row;
            const RayParams& r = S.ray[g];
            int lo = 0, hi = 0;
            if (y >= r.v && y < r.v + s) {
                const int64_t base = int64_t(y) * wp;
                tab(g, L.row_ptr[base + r.u + s] - L.row_ptr[base + r.u]);  // scanned: full window
                int x0, x1;
                if (footprint_row(S.fp[g], QC.C, pad, QC.width, QC.height, r.u, r.v, y, x0, x1)) {
                    lo = L.row_ptr[base + x0];
                    hi = L.row_ptr[base + x1 + 1];
                    if (lo < hi) {
                        atomicMin(&S.slo[row], lo);
                        atomicMax(&S.shi[row], hi);
                    }
                }
            }
            S.rlo[row][g] = lo;
            S.rhi[row][g] = hi;
        }
        __syncthreads();
        for (int row = tid; row < nrows; row += kThreads)
            if (S.slo[row] > S.shi[row]) S.slo[row] = S.shi[row] = 0;  // nothing staged
        __syncthreads();
        // chunk cursor (identical in every thread)
        int row = 0, c0 = S.slo[0];
        auto advance = [&](int& rw, int& cc) {
            cc += kStage;
            while (rw < nrows && cc >= S.shi[rw]) {
                rw++;
                if (rw < nrows) cc = S.slo[rw];
            }
        };
        if (c0 >= S.shi[0]) {  // empty first row(s)
            c0 -= kStage;
            advance(row, c0);
        }
        int buf = 0;
        if (row < nrows) issue(0, c0, min(c0 + kStage, S.shi[row]));
        cp_commit();
        while (row < nrows) {
            int nrow = row, nc0 = c0;
            advance(nrow, nc0);
            if (nrow < nrows) {
                issue(buf ^ 1, nc0, min(nc0 + kStage, S.shi[nrow]));
                cp_commit();
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
            __syncthreads();
            const int c1 = min(c0 + kStage, S.shi[row]);
            for (int g = warp; g < G; g += kWarps) {
                const int lo = max(S.rlo[row][g], c0), hi = min(S.rhi[row][g], c1);
                if (lo < hi) {  // warp-uniform
                    test(buf, g, lo, hi, c0);
                    done(g);  // end of ray g's slots in this chunk
                }
            }
            __syncthreads();
            row = nrow;
            c0 = nc0;
            buf ^= 1;
        }
    }
}


// ---------------------------------------------------------------- pass 1
struct FillSmem {
    GroupHead head;
    float4 pf[2][kStageFill];
    double px[2][kStageFill], py[2][kStageFill], pz[2][kStageFill];
    int pid[2][kStageFill];
    int fill[kGroupMax], scn[kGroupMax];
    unsigned tmin[kGroupMax], tmax[kGroupMax];  // fkey bounds of the accepted t (for the sort)
    int64_t off[kGroupMax];
};


// Pass 1 (the only streaming pass): stream a group's rows and append the
// accepted pairs (t, id, dist), unsorted, to each ray's scratch segment at
// soff[r] (capacity from k_query_bound); write the exact count, probes and
// scanned of every ray.
__global__ void __launch_bounds__(kThreads, HP_SCAN_MINB) k_query_scan(hp_query_layout L, int64_t wp, int pad, Rays R, QCam QC,
                                                         int64_t m, const int64_t* __restrict__ soff,
                                                         int* __restrict__ sc_id, double* __restrict__ sc_t,
                                                         double* __restrict__ sc_d, uint2* __restrict__ tmm,
                                                         int64_t* __restrict__ counts,
                                                         int64_t* __restrict__ probes, int64_t* __restrict__ scanned,
                                                         int64_t capacity) {
    extern __shared__ __align__(16) unsigned char dyn[];
    FillSmem& S = *reinterpret_cast<FillSmem*>(dyn);
    if (soff[m] > capacity) return;  // scratch too small: hp_query_count reports it in offsets[m]
    const int s = 2 * pad + 1;
    const float4* __restrict__ relf = reinterpret_cast<const float4*>(L.relf);
    for (int64_t r0 = int64_t(blockIdx.x) * kGroupMax; r0 < m; r0 += int64_t(gridDim.x) * kGroupMax) {
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        if (threadIdx.x < G) {
            S.fill[threadIdx.x] = 0;
            S.scn[threadIdx.x] = 0;
            S.tmin[threadIdx.x] = 0xffffffffu;
            S.tmax[threadIdx.x] = 0u;
            S.off[threadIdx.x] = soff[r0 + threadIdx.x];
        }
        group_setup(S.head, R, QC, r0, G, s);
        unsigned lmin = 0xffffffffu, lmax = 0u;  // this lane's t bounds for the current ray
        stream_group<kStageFill>(
            S.head, G, L, wp, s, QC,
            [&](int buf, int c0, int c1) {
                for (int k = c0 + int(threadIdx.x); k < c1; k += kThreads) {
                    const int i = k - c0;
                    cp_async16(&S.pf[buf][i], relf + k);
                    cp_async8(&S.px[buf][i], L.rel_x + k);
                    cp_async8(&S.py[buf][i], L.rel_y + k);
                    cp_async8(&S.pz[buf][i], L.rel_z + k);
                    cp_async4(&S.pid[buf][i], L.point_id + k);
                }
            },
            [&](int buf, int g, int lo, int hi, int c0) {
                // the ray's filter terms, output offset and fill count stay in
                // registers for the whole run (shared-memory stores in the loop
                // would otherwise force a re-load per slot)
                const RayParams& r = S.head.ray[g];
                const RayF rf = ray_f(r);
                const int64_t off = S.off[g];
                int fill = S.fill[g];
                for (int base = lo; base < hi; base += 32) {
                    const int k = base + lane_id();
                    int cls = 0;
                    double t = 0.0, d2 = 0.0;
                    if (k < hi) {
                        const int i = k - c0;
                        cls = cone_filter(S.pf[buf][i], rf);
                        if (cls != 0) {
                            const bool ok = cone_test(S.px[buf][i], S.py[buf][i], S.pz[buf][i], r, t, d2);
                            if (cls == 2) cls = ok ? 1 : 0;
                        }
                    }
                    const unsigned b = __ballot_sync(0xffffffffu, cls == 1);
                    if (cls == 1) {
                        const int64_t pos = off + fill + __popc(b & ((1u << lane_id()) - 1));
                        HP_ASSERT(pos < capacity);
                        sc_t[pos] = t;
                        sc_d[pos] = d2;  // dist^2: the sort takes the square root
                        sc_id[pos] = S.pid[buf][k - c0];
                        lmin = min(lmin, fkey(__double2float_rd(t)));
                        lmax = max(lmax, fkey(__double2float_ru(t)));
                    }
                    fill += __popc(b);
                }
                if (lane_id() == 0) S.fill[g] = fill;  // ray g belongs to this warp alone
                __syncwarp();
            },
            [&](int g, int n) { atomicAdd(&S.scn[g], n); },
            [&](int g) {  // per-lane t bounds of ray g's matches in this chunk -> the ray's
                const unsigned lo = __reduce_min_sync(0xffffffffu, lmin);
                const unsigned hi = __reduce_max_sync(0xffffffffu, lmax);
                if (lane_id() == 0) {
                    S.tmin[g] = min(S.tmin[g], lo);
                    S.tmax[g] = max(S.tmax[g], hi);
                }
                lmin = 0xffffffffu;
                lmax = 0u;
            });
        __syncthreads();
        if (threadIdx.x < G) {
            tmm[r0 + threadIdx.x] = make_uint2(S.tmin[threadIdx.x], S.tmax[threadIdx.x]);
            counts[r0 + threadIdx.x] = S.fill[threadIdx.x];
            probes[r0 + threadIdx.x] = int64_t(s) * s;
            scanned[r0 + threadIdx.x] = S.scn[threadIdx.x];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- sort

template <int kCap>
struct SortSmem {
    double t[kCap];
    int id[kCap];  // point ids < 2^31 (hp_build)
    union {
        struct {
            unsigned int bk[kCap];  // fine bucket << 16 | local index
            int hist[kCap + 1];
        };
        double d[kCap];  // dist, loaded once the ranks are known
    };
    unsigned short lst[kCap];
    unsigned short perm[kCap];
    int chist[kCoarse + 1];
    int scan_sh[33];
    int fcount, fbad;  // per-ray facts for the sampler (see sort_segment)
};


// IdT: int32 (the match scratch) or int64 (in place in the output arrays,
// for the parts of split rays: every input is in shared memory before the
// corresponding output is written).
template <int kCap, int kT, class IdT>
__device__ void sort_segment(SortSmem<kCap>& F, int q, uint2 mm, const double* st, const IdT* sid,
                             const double* sd, int64_t* gid, double* gt, double* gd, double slope, int* fact) {
    const int tid = threadIdx.x;
    if (tid == 0) F.fcount = F.fbad = 0;
    // all of the segment's loads in flight at once
    for (int e = tid; e < q; e += kT) {
        cp_async8(&F.t[e], st + e);
        if constexpr (sizeof(IdT) == 4)
            cp_async4(&F.id[e], sid + e);
        else
            F.id[e] = int(sid[e]);
    }
    cp_commit();
    if (q > 64) {
        for (int k = tid; k <= kCoarse; k += kT) F.chist[k] = 0;
        for (int k = tid; k <= q; k += kT) F.hist[k] = 0;
    }
    cp_wait<0>();
    __syncthreads();
    rank_segment<kCap, kT>(q, from_fkey(mm.x), from_fkey(mm.y), F.t, F.id, F.bk, F.hist, F.lst, F.perm, F.chist,
                           F.scan_sh);
    // dist into the (now free) bucket arrays, in flight while t / id go out
    for (int e = tid; e < q; e += kT) cp_async8(&F.d[e], sd + e);
    cp_commit();
    // Facts for the sampler's fast path (hp_sample_run, query_facts): the
    // segment is sorted by construction; record whether every t / dist is
    // finite with dist >= 0, and #{dist <= slope * t_0} (its r_0 count).
    bool bad = false;
    for (int p = tid; p < q; p += kT) {
        const int e = F.perm[p];
        const double te = F.t[e];
        gt[p] = te;
        gid[p] = F.id[e];
        bad |= !(fabs(te) <= DBL_MAX);
    }
    cp_wait<0>();
    __syncthreads();
    if (fact) {
        const double r0 = dmul(slope, F.t[F.perm[0]]);
        int cnt = 0;
        for (int p = tid; p < q; p += kT) {
            const double d = sqrt(F.d[F.perm[p]]);
            gd[p] = d;
            bad |= !(d >= 0.0) || !(d <= DBL_MAX);
            cnt += d <= r0;
        }
        cnt = warp_sum(cnt);
        if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(&F.fbad, 1);
        if (lane_id() == 0 && cnt) atomicAdd(&F.fcount, cnt);
    } else {
        for (int p = tid; p < q; p += kT) gd[p] = sqrt(F.d[F.perm[p]]);
    }
    __syncthreads();
    if (fact && tid == 0) *fact = F.fbad ? -1 : F.fcount;
}

// Size classes of rays to sort (by match count): shared-memory sorts with
// capacities kSortCap (smaller capacity = more resident CTAs), then the rays
// above kSortHuge, split into parts (k_query_split).
constexpr int kSortClasses = 4;
__constant__ int kSortCap[kSortClasses] = {1024, 2048, 4096, 8192};
constexpr int kSortHuge = 8192;  // above: split into t-ordered parts of <= kSortHuge (k_query_split)
__global__ void k_sort_classes(const int64_t* __restrict__ off, int64_t m, int* __restrict__ lists,
                               int* __restrict__ counts) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r - threadIdx.x < m;
         r += int64_t(gridDim.x) * blockDim.x) {
        int cls = -1;
        if (r < m) {
            const int64_t q = off[r + 1] - off[r];
            cls = kSortClasses;
#pragma unroll
            for (int c = kSortClasses - 1; c >= 0; c--)
                if (q <= kSortCap[c]) cls = c;
            if (q == 0) cls = -1;  // nothing to sort
        }
#pragma unroll
        for (int c = 0; c <= kSortClasses; c++) {  // warp-aggregated append
            const unsigned b = __ballot_sync(0xffffffffu, cls == c);
            if (!b) continue;
            int base = 0;
            if (lane_id() == __ffs(b) - 1) base = atomicAdd(&counts[c], __popc(b));
            base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
            if (cls == c) lists[int64_t(c) * m + base + __popc(b & ((1u << lane_id()) - 1))] = int(r);
        }
    }
}

// Sort the rays of one size class (list of ray ids) from the scratch (ray r
// at soff[r]) into the outputs (at off[r]) in shared memory.
template <int kCap, int kT>
__global__ void __launch_bounds__(kT, (kCap == 2048 && kT == 512) ? 4 : 0) k_query_sort(const int64_t* __restrict__ off, const int64_t* __restrict__ soff,
                                                   const uint2* __restrict__ tmm, const double* slopes, int* facts,
                                                   const int* __restrict__ list,
                                                   const int* __restrict__ list_n, double* __restrict__ st,
                                                   int* __restrict__ sid, double* __restrict__ sd,
                                                   int64_t* __restrict__ out_id, double* __restrict__ out_t,
                                                   double* __restrict__ out_d) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = *list_n;
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
        const int64_t r = list[k];
        const int64_t o = off[r], so = soff[r];
        const int64_t q = off[r + 1] - o;
        // (plain loads under the branch: the .nc path may be speculated)
        double slope = 0.0;
        if (facts) slope = __ldcg(slopes + r);
        sort_segment<kCap, kT, int>(*reinterpret_cast<SortSmem<kCap>*>(dyn), int(q), tmm[r], st + so, sid + so,
                                    sd + so, out_id + o, out_t + o, out_d + o, slope, facts ? facts + r : nullptr);
    }
}


// ---------------------------------------------------------------- huge rays
// Rays with more than kSortHuge matches: one CTA per ray splits the ray's
// matches into t-ordered parts of <= kSortHuge (a 2048-bin linear histogram
// of t over the ray's float bounds, bins grouped greedily), scattering them
// into the ray's output segment part by part; every part is then sorted in
// place in shared memory (k_query_sort_parts).  Parts are disjoint, ordered
// t ranges (the bin map is monotone), so sorted parts = sorted ray.  A single
// bin above kSortHuge (near-equal t) becomes a part sorted by a CTA network.
constexpr int kSplitBins = 2048;
constexpr int kSplitThreads = 1024;
constexpr int kMaxParts = 512;

struct Part {
    int64_t start;  // absolute position in the output arrays
    int size;
    unsigned lo, hi;  // fkey bounds of the part's t
};

struct SplitSmem {
    int hist[kSplitBins + 1];
    int cur[kSplitBins];
    unsigned short bin_part[kSplitBins];
    int pstart[kMaxParts + 1];
    unsigned plo[kMaxParts], phi[kMaxParts];
    int scan_sh[33];
    int np, slot;
};

__global__ void __launch_bounds__(kSplitThreads) k_query_split(
    const int64_t* __restrict__ off, const int64_t* __restrict__ soff, const uint2* __restrict__ tmm,
    const int* __restrict__ list, const int* __restrict__ list_n, const double* __restrict__ st,
    const int* __restrict__ sid, const double* __restrict__ sd, int64_t* __restrict__ out_id,
    double* __restrict__ out_t, double* __restrict__ out_d, Part* __restrict__ parts, int* __restrict__ parts_n,
    int parts_cap) {
    extern __shared__ __align__(16) unsigned char dyn[];
    SplitSmem& S = *reinterpret_cast<SplitSmem*>(dyn);
    const int tid = threadIdx.x;
    const int n = *list_n;
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
        const int64_t r = list[k];
        const int64_t o = off[r], so = soff[r];
        const int q = int(off[r + 1] - o);
        const double tlo = double(from_fkey(tmm[r].x)), thi = double(nextafterf(from_fkey(tmm[r].y), CUDART_INF_F));
        const double span = dsub(thi, tlo);
        const double scale = span > 0.0 ? fmin(__ddiv_rn(double(kSplitBins), span), DBL_MAX) : 0.0;
        auto bin = [&](double t) { return min(int(fmin(dmul(dsub(t, tlo), scale), double(kSplitBins))), kSplitBins - 1); };
        for (int b = tid; b <= kSplitBins; b += kSplitThreads) S.hist[b] = 0;
        __syncthreads();
        for (int e = tid; e < q; e += kSplitThreads) {
            const int b = bin(st[so + e]);
            const unsigned peers = __match_any_sync(__activemask(), b);
            if (lane_id() == __ffs(peers) - 1) atomicAdd(&S.hist[b], __popc(peers));
        }
        __syncthreads();
        block_scan_inplace<(kSplitBins + kSplitThreads - 1) / kSplitThreads>(S.hist, kSplitBins, S.scan_sh);
        __syncthreads();
        // parts: bin b joins part floor(start_b / (kSortHuge / 2)) (a part holds
        // at most kSortHuge / 2 + its last bin's matches), renumbered densely
        constexpr int kHalf = kSortHuge / 2;
        int flag[(kSplitBins + kSplitThreads - 1) / kSplitThreads];
#pragma unroll
        for (int k = 0; k < (kSplitBins + kSplitThreads - 1) / kSplitThreads; k++) {
            const int b = tid * ((kSplitBins + kSplitThreads - 1) / kSplitThreads) + k;
            flag[k] = b < kSplitBins && (b == 0 || S.hist[b] / kHalf != S.hist[b - 1] / kHalf);
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < (kSplitBins + kSplitThreads - 1) / kSplitThreads; k++) {
            const int b = tid * ((kSplitBins + kSplitThreads - 1) / kSplitThreads) + k;
            if (b < kSplitBins) S.cur[b] = flag[k];
        }
        __syncthreads();
        int nparts;
        {
            int v[(kSplitBins + kSplitThreads - 1) / kSplitThreads], acc = 0;
#pragma unroll
            for (int k = 0; k < (kSplitBins + kSplitThreads - 1) / kSplitThreads; k++) {
                const int b = tid * ((kSplitBins + kSplitThreads - 1) / kSplitThreads) + k;
                v[k] = b < kSplitBins ? S.cur[b] : 0;
                acc += v[k];
            }
            int run = block_excl_scan<int>(acc, S.scan_sh, &nparts);
#pragma unroll
            for (int k = 0; k < (kSplitBins + kSplitThreads - 1) / kSplitThreads; k++) {
                const int b = tid * ((kSplitBins + kSplitThreads - 1) / kSplitThreads) + k;
                run += v[k];
                if (b < kSplitBins) {
                    const int p = min(run - 1, kMaxParts - 1);
                    S.bin_part[b] = (unsigned short)p;
                    if (v[k] && run - 1 < kMaxParts) {
                        S.pstart[p] = S.hist[b];
                        // t bounds of the part from its first bin's lower edge (any
                        // bounds keep the part sort's bucket map monotone)
                        S.plo[p] = fkey(__double2float_rd(tlo + double(b) / scale));
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            const int np = min(nparts, kMaxParts);
            S.np = np;
            S.pstart[np] = q;
            S.slot = atomicAdd(parts_n, np);
        }
        __syncthreads();
        for (int p = tid; p < S.np; p += kSplitThreads) S.phi[p] = p + 1 < S.np ? S.plo[p + 1] : tmm[r].y;
        for (int b = tid; b < kSplitBins; b += kSplitThreads) S.cur[b] = S.hist[b];
        __syncthreads();
        for (int e = tid; e < q; e += kSplitThreads) {
            const double t = st[so + e];
            const int b = bin(t);
            const unsigned peers = __match_any_sync(__activemask(), b);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (lane_id() == leader) base = atomicAdd(&S.cur[b], __popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int pos = base + __popc(peers & ((1u << lane_id()) - 1));
            out_t[o + pos] = t;
            out_id[o + pos] = sid[so + e];
            out_d[o + pos] = sd[so + e];  // dist^2 until the part sort
        }
        __syncthreads();
        for (int p = tid; p < S.np; p += kSplitThreads) {
            const int slot = S.slot + p;
            if (slot < parts_cap)
                parts[slot] = Part{o + S.pstart[p], S.pstart[p + 1] - S.pstart[p], S.plo[p], S.phi[p]};
        }
        __syncthreads();
    }
}

// Sort the parts in place in the output arrays: shared memory for parts of
// <= kCap, a CTA sorting network in global memory for the larger ones.
template <int kCap, int kT>
__global__ void __launch_bounds__(kT) k_query_sort_parts(const Part* __restrict__ parts,
                                                         const int* __restrict__ parts_n, int parts_cap,
                                                         int64_t* out_id, double* out_t, double* out_d) {
    extern __shared__ __align__(16) unsigned char dyn[];
    const int n = min(*parts_n, parts_cap);
    for (int k = blockIdx.x; k < n; k += gridDim.x) {
        const Part P = parts[k];
        int64_t* ii = out_id + P.start;
        double* tt = out_t + P.start;
        double* dd = out_d + P.start;
        if (P.size <= kCap) {
            sort_segment<kCap, kT, int64_t>(*reinterpret_cast<SortSmem<kCap>*>(dyn), P.size,
                                            make_uint2(P.lo, P.hi), tt, ii, dd, ii, tt, dd, 0.0, nullptr);
        } else {
            block_bitonic_sort(
                P.size, [&](int64_t a, int64_t b) { return key_less(tt[a], ii[a], tt[b], ii[b]); },
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
            for (int64_t p = threadIdx.x; p < P.size; p += kT) dd[p] = sqrt(dd[p]);  // dist^2 -> dist
            __syncthreads();
        }
    }
}


}  // namespace
}  // namespace hp

using namespace hp;

// workspace: scan scratch | scratch offsets soff [m+1] | per-ray float t
// bounds | ray lists of the sort size classes | class counts | unsorted
// matches (t, id, dist) x capacity
struct QueryWs {
    void* scan;
    int64_t* soff;
    uint2* tmm;
    int* lists;
    int* counts;
    double* st;
    int* sid;
    double* sd;
    Part* parts;  // t-ordered parts of the rays above kSortHuge
    int* parts_n;
    int parts_cap;
};

struct SortArgs {
    const int64_t* offsets;
    QueryWs w;
    int64_t m;
    int64_t* ids;
    double* t;
    double* d;
    const double* slopes;
    int* facts;
};

// One shared-memory size class: grid = SMs x resident CTAs (occupancy API).
template <int kCap, int kT>
static int launch_sort(const SortArgs& A, int cls, cudaStream_t s) {
    // once per process (thread-safe initialisation); a failure shows at launch
    const int occ = kernel_occupancy((const void*)k_query_sort<kCap, kT>, kT, sizeof(SortSmem<kCap>));
    if (occ < 0) return occ;
    k_query_sort<kCap, kT><<<device_sms() * occ, kT, sizeof(SortSmem<kCap>), s>>>(
        A.offsets, A.w.soff, A.w.tmm, A.slopes, A.facts, A.w.lists + int64_t(cls) * A.m, A.w.counts + cls, A.w.st, A.w.sid, A.w.sd,
        A.ids, A.t, A.d);
    HP_CHECK_LAUNCH("k_query_sort");
    return HP_OK;
}


static QueryWs carve_query(Carver& c, int64_t m, int64_t cap) {
    QueryWs w;
    w.scan = c.take<char>(scan_workspace_bytes(m + 1));
    w.soff = c.take<int64_t>(m + 1);
    w.tmm = c.take<uint2>(m > 0 ? m : 1);
    w.lists = c.take<int>((kSortClasses + 1) * (m > 0 ? m : 1));
    w.counts = c.take<int>(64);
    w.st = c.take<double>(cap > 0 ? cap : 1);
    w.sid = c.take<int>(cap > 0 ? cap : 1);
    w.sd = c.take<double>(cap > 0 ? cap : 1);
    // parts: consecutive parts of a ray hold > kSortHuge matches together
    const int64_t pc = 2 * (cap > 0 ? cap : 0) / kSortHuge + m + 64;
    w.parts_cap = int(pc < INT_MAX ? pc : INT_MAX);
    w.parts = c.take<Part>(w.parts_cap);
    w.parts_n = c.take<int>(1);
    return w;
}

extern "C" int hp_query_workspace_bytes(int64_t m, int64_t pad, int64_t capacity, size_t* bytes) {
    Carver c(nullptr, 0);
    carve_query(c, m, capacity);
    *bytes = c.used + 256;
    (void)pad;
    return HP_OK;
}

extern "C" int hp_query_count(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                              int64_t pad, const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                              const double* t_near, const double* t_far, const double* slopes, int64_t m,
                              int64_t* offsets, int64_t* probes, int64_t* scanned, int64_t capacity,
                              void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(check_common(layout, pad, m, padded_w, padded_h));
    Carver cv(workspace, workspace_bytes);
    QueryWs w = carve_query(cv, m, capacity);
    if (!cv.ok()) {
        set_error("hp_query_count: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    const QCam QC = make_qcam(cam);
    if (m > 0) {
        {
            TimedSpan ts("k_query_bound", s);
            k_query_bound<<<group_grid(m, 8), kThreads, 0, s>>>(layout, padded_w, int(pad), R, QC, m, w.soff);
            HP_CHECK_LAUNCH("k_query_bound");
        }
        HP_TRY(exclusive_scan_i64(w.soff, w.soff, m, w.scan, s));
        const int occ = kernel_occupancy((const void*)k_query_scan, kThreads, sizeof(FillSmem));
        if (occ < 0) return occ;
        TimedSpan ts("k_query_scan", s);
        k_query_scan<<<group_grid(m, HP_SCAN_MINB ? HP_SCAN_MINB : 4), kThreads, sizeof(FillSmem), s>>>(layout, padded_w, int(pad), R, QC, m, w.soff,
                                                                         w.sid, w.st, w.sd, w.tmm, offsets, probes,
                                                                         scanned, capacity);
        HP_CHECK_LAUNCH("k_query_scan");
    }
    HP_TRY(exclusive_scan_i64(offsets, offsets, m, w.scan, s));
    if (m > 0) {
        k_mark_overflow<<<1, 1, 0, s>>>(w.soff + m, capacity, offsets + m);
        HP_CHECK_LAUNCH("k_mark_overflow");
    }
    return HP_OK;
}

extern "C" int hp_query_fill(const int64_t* offsets, int64_t m, int64_t total, int64_t* ids, double* t_proj,
                             double* dist_perp, const double* slopes, int32_t* facts, int64_t capacity,
                             void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    if (m < 0 || total < 0) {
        set_error("hp_query_fill: invalid arguments");
        return HP_EINVAL;
    }
    if (facts && !slopes) {
        set_error("hp_query_fill: facts need the query's slopes");
        return HP_EINVAL;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (facts && m > 0 && cudaMemsetAsync(facts, 0xff, size_t(m) * sizeof(int32_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_query_fill memset");  // -1: unknown
    if (m == 0 || total == 0) return HP_OK;
    Carver cv(workspace, workspace_bytes);
    QueryWs w = carve_query(cv, m, capacity);
    if (!cv.ok()) {
        set_error("hp_query_fill: workspace too small");
        return HP_ESPACE;
    }
    if (cudaMemsetAsync(w.counts, 0, (kSortClasses + 1) * sizeof(int), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_query_fill memset");
    k_sort_classes<<<grid_for(m, 256), 256, 0, s>>>(offsets, m, w.lists, w.counts);
    HP_CHECK_LAUNCH("k_sort_classes");
    const SortArgs A{offsets, w, m, ids, t_proj, dist_perp, slopes, facts};
    {
        TimedSpan ts("k_query_sort", s);
        HP_TRY((launch_sort<1024, kThreads>(A, 0, s)));
        HP_TRY((launch_sort<2048, 512>(A, 1, s)));
    }
    TimedSpan ts("k_query_sort_large", s);
    HP_TRY((launch_sort<4096, 512>(A, 2, s)));
    {
        TimedSpan t8("k_query_sort_8192", s);
        HP_TRY((launch_sort<kSortHuge, 1024>(A, 3, s)));
    }
    // rays above kSortHuge: split into t-ordered parts, sort the parts in place
    const int occ_split = kernel_occupancy((const void*)k_query_split, kSplitThreads, sizeof(SplitSmem));
    if (occ_split < 0) return occ_split;
    const int occ_parts =
        kernel_occupancy((const void*)k_query_sort_parts<kSortHuge, 1024>, 1024, sizeof(SortSmem<kSortHuge>));
    if (occ_parts < 0) return occ_parts;
    if (cudaMemsetAsync(w.parts_n, 0, sizeof(int), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_query_fill memset");
    TimedSpan tsp("k_query_split", s);
    k_query_split<<<device_sms(), kSplitThreads, sizeof(SplitSmem), s>>>(
        offsets, w.soff, w.tmm, w.lists + kSortClasses * m, w.counts + kSortClasses, w.st, w.sid, w.sd, ids, t_proj,
        dist_perp, w.parts, w.parts_n, w.parts_cap);
    HP_CHECK_LAUNCH("k_query_split");
    k_query_sort_parts<kSortHuge, 1024><<<device_sms() * occ_parts, 1024, sizeof(SortSmem<kSortHuge>), s>>>(
        w.parts, w.parts_n, w.parts_cap, ids, t_proj, dist_perp);
    HP_CHECK_LAUNCH("k_query_sort_parts");
    return HP_OK;
}

extern "C" int hp_query_bounds(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                               int64_t pad, const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                               const double* t_near, const double* t_far, const double* slopes, int64_t m,
                               int64_t* bound_off, void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(check_common(layout, pad, m, padded_w, padded_h));
    if (workspace_bytes < scan_workspace_bytes(m + 1)) {
        set_error("hp_query_bounds: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (m > 0) {
        const Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
        const QCam QC = make_qcam(cam);
        TimedSpan ts("k_query_bound", s);
        k_query_bound<<<group_grid(m, 8), kThreads, 0, s>>>(layout, padded_w, int(pad), R, QC, m, bound_off);
        HP_CHECK_LAUNCH("k_query_bound");
    }
    HP_TRY(exclusive_scan_i64(bound_off, bound_off, m, workspace, s));
    return HP_OK;
}

