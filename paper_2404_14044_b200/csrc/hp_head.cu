// hp_head.cu — the query for callers that only want samples: per ray, the
// head of its matches in (t, id) order, without materialising its full match
// list.
//
// Reference: the chained hash_query_batch (_kernels.py:86-157; cone test
// :22-36, canonical order :39-73) -> sample_batch (:552-700) of the renderer
// (renderer.py:119-124).  The sampler only ever reads a head of each ray's t
// order (hp_sample.cu, prefix mode), so the query keeps, per accepted
// (ray, point) pair, 8 bytes -- a lower bound of the exact t as an
// order-preserving float key and the pair's layout slot -- instead of the
// 20-byte exact (t, id, dist) record, and recomputes the exact values only for
// the head, from the L2-resident layout, with the reference's own expression
// (bit-identical: cone_t / cone_dist2 of hp_cone.cuh).
//
//   k_head_scan    the streaming pass: a CTA claims a group of <= 32 adjacent
//                  rays, places their scratch segments (each ray's footprint
//                  slot count, one cursor atomic per group) and streams the
//                  union of their footprint rows through
//                  shared memory, fp32 copies only (16 B per point), staged by
//                  1-D bulk copies (cp.async.bulk + mbarrier); the fp32 filter
//                  settles almost every pair; the few uncertain pairs are
//                  deferred per warp and decided in batches by the exact fp64
//                  test (coordinates gathered from rel4).  Accepted pairs ->
//                  (key, slot) appended to the ray's scratch segment.
//   k_head_classes / k_head_select (long rays: warp per ray, key histogram ->
//                  the key cut K_c) / k_head_sort (one CTA per ray: stage the
//                  selected slots, gather + exact t / dist^2, trim the band
//                  above the cut, exact (t, id) rank, write the head).
//
// Exactness (DESIGN.md §6 "Heads"): every key is a lower bound of its pair's
// exact t (sure accepts: RD(t32 - eps) with |t32 - t64| <= eps; fp64-decided
// pairs: RD(t64)).  A long ray keeps the pairs with key <= K_c whose exact t is
// below T_c = float(K_c + 1); every pair left out has t >= T_c (key > K_c, or
// trimmed), so the head is exactly a prefix of the ray's (t, id) order.  The
// cuts handed to the sampler are lower bounds of the left-out t and dist
// (hp_sample.cu only relies on "every left-out t >= cut_t, dist >= cut_d").
#include "hp_query_core.cuh"
#include "hp_sample_core.cuh"

namespace hp {
namespace {

constexpr int kHeadCap = 1024;   // longest head; rays up to this are sorted whole
constexpr int kHeadLong = 4096;  // the long-head mode (a later chance for rays 1024 do not cover)
constexpr int kHeadMid = 2048;   // long-head mode: heads up to this in a denser CTA configuration
constexpr int kHeadSmall = 512;  // rays up to this: a smaller, denser CTA configuration
#ifndef HP_HEAD_STAGE
#define HP_HEAD_STAGE 1024
#endif
constexpr int kStage = HP_HEAD_STAGE;  // slots per staged chunk (16 B each)
constexpr int kMaxPieces = 8;          // row pieces per chunk
#ifndef HP_HEAD_MINB
#define HP_HEAD_MINB 4
#endif
#ifndef HP_HEAD_SORT_MINB
#define HP_HEAD_SORT_MINB 6
#endif
#ifndef HP_HEAD_U_MAX
#define HP_HEAD_U_MAX 384  // bound factors precomputed for the first this many head entries
#endif
#ifndef HP_SCAN_DYN
#define HP_SCAN_DYN 1  // k_head_scan: a chunk's rays claimed by the warps one at a time
#endif
#ifndef HP_SELECT_U
#define HP_SELECT_U 8  // keys (and slots) per lane in flight in k_head_select
#endif

// ---------------------------------------------------------------- bulk copies
__device__ __forceinline__ unsigned smem_u32(const void* p) { return unsigned(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n HP_MBAR_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra HP_MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() { return (1u << lane_id()) - 1u; }

// ---------------------------------------------------------------- scan
// stream_group (hp_query.cu) with the chunks staged by bulk copies: thread 0
// packs a chunk from consecutive rows' staged ranges ("pieces"), arms the
// buffer's mbarrier and issues one bulk copy per piece; every thread waits on
// the barrier's phase (tracked in `phase`, bit b = parity of buffer b's next
// completion).  Chunk i + 1 is in flight while chunk i is tested; a warp takes
// each of its rays through all of a chunk's pieces (`chunk`).  `tab` counts
// the slots of each ray's full window row (the scanned output).
template <class Issue, class Chunk, class Tab>
__device__ void stream_group_bulk(GroupHead& S, uint64_t* bar, int4 (*pieces)[kMaxPieces], int* npieces,
                                  int* ctr, unsigned& phase, int G, const hp_query_layout L, int64_t wp, int s,
                                  const QCam& QC, Issue issue, Chunk chunk, Tab tab) {
    const int tid = threadIdx.x, warp = warp_id();
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
        // Chunks of up to kStage slots packed from consecutive rows' staged
        // ranges ("pieces"; a row longer than the space left is split), so a
        // chunk barrier covers several rows of work.  Thread 0 plans chunk
        // i + 1 (its pieces in shared memory, one bulk copy per piece on the
        // buffer's mbarrier) while chunk i is tested.
        int prow = 0, pc = S.slo[0];  // thread 0's cursor: next slot to stage
        auto plan_issue = [&](int b) {
            int n = 0, off = 0;
            while (prow < nrows && n < kMaxPieces && off < kStage) {
                if (pc >= S.shi[prow]) {
                    if (++prow < nrows) pc = S.slo[prow];
                    continue;
                }
                const int take = min(S.shi[prow] - pc, kStage - off);
                pieces[b][n] = make_int4(prow, pc, pc + take, off);
                n++;
                off += take;
                pc += take;
            }
            npieces[b] = n;
            ctr[b] = 0;  // nobody reads it: the chunk that used it ended at a barrier
            if (n) {
                mbar_arrive_tx(&bar[b], unsigned(off) * 16u);
                for (int i = 0; i < n; i++) issue(b, pieces[b][i].w, pieces[b][i].y, pieces[b][i].z);
            }
        };
        int buf = 0;
        if (tid == 0) plan_issue(0);
        __syncthreads();
        while (npieces[buf] > 0) {
            if (tid == 0) plan_issue(buf ^ 1);
            mbar_wait(&bar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
            // ray-major: a warp takes each of its rays through all of the
            // chunk's pieces (rows), its per-ray state loaded once per chunk
            const int np = npieces[buf];
#if HP_SCAN_DYN
            // rays handed out one at a time (their footprints differ: a static
            // split leaves warps waiting at the chunk barrier)
            for (;;) {
                int g = 0;
                if (lane_id() == 0) g = atomicAdd(&ctr[buf], 1);
                g = __shfl_sync(0xffffffffu, g, 0);
                if (g >= G) break;
                chunk(buf, g, np, pieces[buf]);
            }
#else
            for (int g = warp; g < G; g += kWarps) chunk(buf, g, np, pieces[buf]);
#endif
            __syncthreads();  // buffer `buf` is refilled two chunks later; npieces[buf ^ 1] is visible
            buf ^= 1;
        }
        __syncthreads();  // every thread has read npieces before the next batch plans over it
    }
}

struct HeadScanSmem {
    GroupHead head;
    float4 pf[2][kStage];
    uint64_t bar[2];
    int4 pieces[2][kMaxPieces];  // (row, a, b, smem offset) of each buffer's chunk
    int npieces[2];
    int ctr[2];          // each buffer's next ray (HP_SCAN_DYN)
    int fill[kGroupMax], scn[kGroupMax], bad[kGroupMax];
    unsigned kmin[kGroupMax], kmax[kGroupMax];
    int64_t off[kGroupMax], end[kGroupMax];
    int dq[kWarps][64];  // deferred (uncertain) slots of the warp's current ray run
    int64_t next;        // the CTA's current group (claimed from the work counter)
    int bnd[kGroupMax];  // the group's per-ray scratch bounds (footprint slots)
    int skip;            // the group's scratch did not fit the capacity
};

// Per-ray results of the scan: key bounds of the accepted pairs, and whether
// an fp64-decided pair had a non-finite t or dist^2 (the sampler's facts).
struct RayMeta {
    unsigned kmin, kmax;
    int bad, pad_;
};

__global__ void __launch_bounds__(kThreads, HP_HEAD_MINB)
    k_head_scan(hp_query_layout L, int64_t wp, int pad, Rays R, QCam QC, int64_t m, int64_t* __restrict__ soff,
                unsigned* __restrict__ sc_key, int* __restrict__ sc_slot, RayMeta* __restrict__ meta,
                int64_t* __restrict__ counts, int64_t* __restrict__ hcount, int64_t* __restrict__ probes,
                int64_t* __restrict__ scanned, int64_t capacity, unsigned long long* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char dyn[];
    HeadScanSmem& S = *reinterpret_cast<HeadScanSmem*>(dyn);
    const int s = 2 * pad + 1;
    const int lane = lane_id(), warp = warp_id();
    const double4* __restrict__ rel4 = reinterpret_cast<const double4*>(L.rel4);
    if (threadIdx.x == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    unsigned phase = 0;
    // groups of kGroupMax rays claimed dynamically (their costs differ widely:
    // a static split leaves a long tail on small frames / row bands)
    for (;;) {
        if (threadIdx.x == 0) S.next = int64_t(atomicAdd(work, 1ull)) * kGroupMax;
        __syncthreads();
        const int64_t r0 = S.next;
        if (r0 >= m) break;
        const int G = int(m - r0 < kGroupMax ? m - r0 : kGroupMax);
        if (threadIdx.x < G) {
            S.fill[threadIdx.x] = 0;
            S.scn[threadIdx.x] = 0;
            S.bad[threadIdx.x] = 0;
            S.kmin[threadIdx.x] = 0xffffffffu;
            S.kmax[threadIdx.x] = 0u;
            S.bnd[threadIdx.x] = 0;
        }
        group_setup(S.head, R, QC, r0, G, s);
        // each ray's scratch segment: its bound (the footprint slots the
        // stream below tests, as k_query_bound counts them), placed by one
        // atomic per group on the scratch cursor work[3] (which ends at the
        // total the frame needs, also when it exceeds the capacity)
        for (int idx = threadIdx.x; idx < s * G; idx += kThreads) {
            const int row = idx / G, g = idx - row * G;
            const RayParams& r = S.head.ray[g];
            const int y = r.v + row;
            int x0, x1;
            if (footprint_row(S.head.fp[g], QC.C, pad, QC.width, QC.height, r.u, r.v, y, x0, x1)) {
                const int64_t base = int64_t(y) * wp;
                const int n = L.row_ptr[base + x1 + 1] - L.row_ptr[base + x0];
                if (n > 0) atomicAdd(&S.bnd[g], n);
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int b = lane < G ? S.bnd[lane] : 0;
            const int inc = warp_incl_scan(b);
            const int tot = __shfl_sync(0xffffffffu, inc, 31);
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(work + 3, (unsigned long long)tot);
            base = __shfl_sync(0xffffffffu, base, 0);
            if (lane < G) {
                S.off[lane] = int64_t(base) + inc - b;
                S.end[lane] = int64_t(base) + inc;
                soff[r0 + lane] = int64_t(base) + inc - b;
            }
            if (lane == 0) S.skip = int64_t(base) + tot > capacity;
        }
        __syncthreads();
        if (S.skip) continue;  // the frame is re-run with the reported size; S.next is rewritten after a barrier
        stream_group_bulk(
            S.head, S.bar, S.pieces, S.npieces, S.ctr, phase, G, L, wp, s, QC,
            [&](int buf, int off, int c0, int c1) {  // one piece: slots [c0, c1) to pf[buf][off..]
                bulk_g2s(&S.pf[buf][off], L.relf + 4 * int64_t(c0), unsigned(c1 - c0) * 16u, &S.bar[buf]);
            },
            [&](int buf, int g, int np, const int4* pcs) {  // ray g over the chunk's pieces
                // lane i < np: ray g's sub-range of piece i (row, a, b, smem offset); the
                // touched pieces are then walked from the ballot
                int plo = 0, phi = 0, pc0 = 0;
                if (lane < np) {
                    const int4 pc = pcs[lane];
                    plo = max(S.head.rlo[pc.x][g], pc.y);
                    phi = min(S.head.rhi[pc.x][g], pc.z);
                    pc0 = pc.y - pc.w;
                }
                const unsigned touched = __ballot_sync(0xffffffffu, plo < phi);
                if (!touched) return;  // warp-uniform
                const RayParams& rp = S.head.ray[g];
                const RayF rf = ray_f(rp);
                const int64_t off = S.off[g];
                unsigned* __restrict__ kout = sc_key + off;  // ray g's scratch segment
                int* __restrict__ sout = sc_slot + off;
                const unsigned below = lanemask_lt();
                int fill = S.fill[g];
                int* dq = S.dq[warp];
                int nq = 0;  // deferred pairs (warp-uniform)
                unsigned lmin = 0xffffffffu, lmax = 0u;  // this lane's key bounds for ray g
                int lbad = 0;
                // the deferred pairs, 32 at a time on all lanes: gather the exact
                // coordinates, the reference's fp64 test, append the accepted
                auto flush = [&](int n) {
                    __syncwarp();
                    int k = -1;
                    bool ok = false;
                    double t = 0.0, d2 = 0.0;
                    if (lane < n) {
                        k = dq[lane];
                        const double4 a = rel4[k];
                        ok = cone_test(a.x, a.y, a.z, rp, t, d2);
                    }
                    const unsigned b = __ballot_sync(0xffffffffu, ok);
                    if (ok) {
                        const int pos = fill + __popc(b & below);
                        HP_ASSERT(off + pos < S.end[g]);
                        const unsigned key = fkey(__double2float_rd(t));
                        kout[pos] = key;
                        sout[pos] = k;
                        lmin = min(lmin, key);
                        lmax = max(lmax, key);
                        lbad |= !(fabs(t) <= DBL_MAX) || !(d2 <= DBL_MAX);
                    }
                    fill += __popc(b);
                    __syncwarp();
                    if (n < nq && lane < nq - n) dq[lane] = dq[n + lane];  // the rest (< 32) to the front
                    __syncwarp();
                    nq -= n;
                };
                for (unsigned tm = touched; tm; tm &= tm - 1) {
                    const int i = __ffs(tm) - 1;
                    const int lo = __shfl_sync(0xffffffffu, plo, i), hi = __shfl_sync(0xffffffffu, phi, i);
                    const int c0 = __shfl_sync(0xffffffffu, pc0, i);
                    for (int base = lo; base < hi; base += 32) {
                        const int k = base + lane;
                        int cls = 0;
                        float tf = 0.0f, eps = 0.0f;
                        if (k < hi) cls = cone_filter_te(S.pf[buf][k - c0], rf, tf, eps);
                        const unsigned acc = __ballot_sync(0xffffffffu, cls == 1);
                        if (cls == 1) {
                            const int pos = fill + __popc(acc & below);
                            HP_ASSERT(off + pos < S.end[g]);
                            const unsigned key = fkey(__fsub_rd(tf, eps));
                            kout[pos] = key;
                            sout[pos] = k;
                            lmin = min(lmin, key);
                            lmax = max(lmax, key);
                        }
                        fill += __popc(acc);
                        const unsigned unc = __ballot_sync(0xffffffffu, cls == 2);
                        if (unc) {
                            HP_ASSERT(nq + __popc(unc) <= 64);
                            if (cls == 2) dq[nq + __popc(unc & below)] = k;
                            nq += __popc(unc);
                            if (nq >= 32) flush(32);
                        }
                    }
                }
                if (nq > 0) flush(nq);
                const unsigned klo = __reduce_min_sync(0xffffffffu, lmin);
                const unsigned khi = __reduce_max_sync(0xffffffffu, lmax);
                const bool anybad = __any_sync(0xffffffffu, lbad);
                if (lane == 0) {  // ray g belongs to this warp alone
                    S.fill[g] = fill;
                    S.kmin[g] = min(S.kmin[g], klo);
                    S.kmax[g] = max(S.kmax[g], khi);
                    if (anybad) S.bad[g] = 1;
                }
                __syncwarp();
            },
            [&](int g, int n) { atomicAdd(&S.scn[g], n); });
        __syncthreads();
        if (threadIdx.x < G) {
            const int64_t r = r0 + threadIdx.x;
            const int q = S.fill[threadIdx.x];
            meta[r] = RayMeta{S.kmin[threadIdx.x], S.kmax[threadIdx.x], S.bad[threadIdx.x], 0};
            counts[r] = q;
            hcount[r] = q < kHeadCap ? q : kHeadCap;
            probes[r] = int64_t(s) * s;
            scanned[r] = S.scn[threadIdx.x];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- classes
// Rays whose head is taken whole (q <= whole): list 0 when q <= kHeadSmall
// (the small sort configuration), else list 1; rays to cut (q > whole):
// list 2, which k_head_select distributes to lists 0 / 1 by the size of the
// head it selects.  The empty rays' outputs are written here.
// With `rays`, output i stands for ray rays[i] (a re-sort of a subset).
__global__ void k_head_classes(const int64_t* __restrict__ off, const int* __restrict__ rays, int64_t m, int whole,
                               int small, int* __restrict__ lists, int* __restrict__ counts, int* __restrict__ plen,
                               int* __restrict__ facts, double* __restrict__ cut_t, double* __restrict__ cut_d,
                               const int64_t* __restrict__ total) {
    // the count pass ran short of scratch (offsets[m] < 0, the caller re-runs
    // it): every head empty, nothing sorted (its counts are not all written)
    const bool over = *total < 0;
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r - threadIdx.x < m;
         r += int64_t(gridDim.x) * blockDim.x) {
        int cls = -1;
        if (r < m) {
            const int64_t ri = rays ? rays[r] : r;
            const int64_t q = over ? 0 : off[ri + 1] - off[ri];
            cls = q == 0 ? -1 : (q > whole ? 2 : (q <= small ? 0 : 1));
            if (q == 0) {
                plen[r] = 0;
                facts[r] = -1;
                cut_t[r] = cut_d[r] = CUDART_INF;
            }
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
            const unsigned b = __ballot_sync(0xffffffffu, cls == c);
            if (!b) continue;
            int base = 0;
            if (lane_id() == __ffs(b) - 1) base = atomicAdd(&counts[c], __popc(b));
            base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
            if (cls == c) lists[int64_t(c) * m + base + __popc(b & lanemask_lt())] = int(r);
        }
    }
}

// ---------------------------------------------------------------- selection
// Rays of more than kHeadCap matches, one warp per ray (a plain stream over
// the 4-byte keys, many rays in flight): a histogram of the keys over
// [kmin, kmax] in bins of 2^sh consecutive keys (the smallest sh giving at
// most kBins bins) -> the first bin b where the running count reaches `want`
// (b - 1 if that bin alone would overflow kHeadCap) -> the key cut K_c = the
// largest key of bin b: sel[r] = (K_c, #{key <= K_c}).  No cut (b < 0):
// K_c = kmin - 1, count 0.
template <int kBins>
__global__ void __launch_bounds__(128) k_head_select(const int64_t* __restrict__ off, const int* __restrict__ rays,
                                                     const int64_t* __restrict__ soff,
                                                     const RayMeta* __restrict__ meta, int want, int whole,
                                                     int cap, int small, const unsigned* __restrict__ sc_key,
                                                     const int* __restrict__ sc_slot, const int64_t* __restrict__ hoff,
                                                     int* __restrict__ stage, uint4* __restrict__ sel,
                                                     const int* __restrict__ list, const int* __restrict__ list_n,
                                                     int* __restrict__ lists, int* __restrict__ counts, int64_t m) {
    __shared__ int hist[4][kBins];
    int* H = hist[warp_id()];
    const int lane = lane_id();
    const int64_t nr = *list_n;
    const int64_t warps = int64_t(gridDim.x) * 4;  // (static: a dynamic claim measured slower here)
    for (int64_t k = int64_t(blockIdx.x) * 4 + warp_id(); k < nr; k += warps) {
        const int64_t i = list[k], r = rays ? rays[i] : i;  // output i, ray r
        const int q = int(off[r + 1] - off[r]);
        if (q <= whole) continue;
        const int64_t so = soff[r];
        const RayMeta M = meta[r];
        const unsigned span1 = M.kmax - M.kmin;  // span - 1
        int sh = 0;
        while ((span1 >> sh) >= unsigned(kBins)) sh++;
        for (int b = lane; b < kBins; b += 32) H[b] = 0;
        __syncwarp();
        constexpr int kU = HP_SELECT_U;
        for (int e0 = 0; e0 < q; e0 += 32 * kU) {  // kU loads per lane in flight
            unsigned kv[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const int e = e0 + u * 32 + lane;
                kv[u] = e < q ? sc_key[so + e] : 0u;
            }
#pragma unroll
            for (int u = 0; u < kU; u++)
                if (e0 + u * 32 + lane < q) {
                    HP_ASSERT(kv[u] >= M.kmin && ((kv[u] - M.kmin) >> sh) < unsigned(kBins));
                    atomicAdd(&H[(kv[u] - M.kmin) >> sh], 1);
                }
        }
        __syncwarp();
        constexpr int kPer = kBins / 32;  // lane owns bins [lane * kPer, lane * kPer + kPer)
        int sum = 0;
#pragma unroll 8
        for (int b = 0; b < kPer; b++) sum += H[lane * kPer + b];
        const int incl = warp_incl_scan(sum);
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= want);
        const int owner = __ffs(hit) - 1;  // exists: q > whole >= want
        unsigned kcut = 0;
        int cnt = 0;
        if (lane == owner) {
            int c = incl - sum, b = lane * kPer;
            for (int j = 0; j < kPer; j++) {
                c += H[lane * kPer + j];
                if (c >= want) {
                    b = lane * kPer + j;
                    break;
                }
            }
            if (c > cap) {  // that bin alone overflows: stop before it
                c -= H[b];
                b -= 1;
            }
            // largest key of bin b (keys above kmax do not occur)
            const unsigned long long kc = (unsigned long long)M.kmin + ((unsigned long long)(b + 1) << sh) - 1ull;
            kcut = unsigned(kc < M.kmax ? kc : M.kmax);
            cnt = c;
        }
        kcut = __shfl_sync(0xffffffffu, kcut, owner);
        cnt = __shfl_sync(0xffffffffu, cnt, owner);
        // the selected pairs' slots, compacted into the ray's head storage (the
        // head sort stages them from there: every cut ray then stages like a
        // whole one); the smallest key left out
        int* st = stage + hoff[i];
        int n = 0;
        unsigned kout = 0xffffffffu;
        for (int e0 = 0; e0 < q; e0 += 32 * kU) {  // keys (L2-warm) and slots, kU of each per lane in flight
            unsigned kv[kU];
            int sv[kU];
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const int e = e0 + u * 32 + lane;
                kv[u] = e < q ? sc_key[so + e] : 0xffffffffu;
                sv[u] = e < q ? __ldcs(sc_slot + so + e) : 0;
            }
#pragma unroll
            for (int u = 0; u < kU; u++) {
                const int e = e0 + u * 32 + lane;
                const bool in = e < q && kv[u] <= kcut;
                if (e < q && !in) kout = min(kout, kv[u]);
                const unsigned bb = __ballot_sync(0xffffffffu, in);
                if (in) st[n + __popc(bb & lanemask_lt())] = sv[u];
                n += __popc(bb);
            }
        }
        kout = __reduce_min_sync(0xffffffffu, kout);
        HP_ASSERT(n == cnt);
        if (lane == 0) {
            sel[i] = make_uint4(kcut, unsigned(cnt), kout, 0u);
            const int cls = cnt <= small ? 0 : 1;  // the sort configuration of this head
            lists[int64_t(cls) * m + atomicAdd(&counts[cls], 1)] = int(i);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- head sort
template <int kCap>
struct HeadSmem {
    double t[kCap];
    double d2[kCap];
    int id[kCap];
    union {
        int slot[kCap];    // staged slots (read before the ranking)
        unsigned bk[kCap]; // rank_segment's bucket words
    };
    int hist[kCap + 1];
    unsigned short lst[kCap], perm[kCap];
    int chist[kCoarse + 1];
    int scan_sh[33];
    unsigned long long cut_d2;         // order key of the trimmed pairs' smallest dist^2
    unsigned kout, thi;                // smallest left-out key; fkey of the largest float(t) staged
    int cnt, keep, fcount, fbad;
    int next;                          // the CTA's current list entry (claimed from the work counter)
};

// One CTA per ray: a ray of <= kCap matches is staged whole (its slots by
// cp.async); a longer one streams its keys and stages the slots of the pairs
// with key <= K_c.  Then the exact t / dist^2 of every staged pair from its
// rel4 record (the reference's expression), the long rays' trim (t >= T_c
// moves to the left-out side), the exact (t, id) rank, and the write-out of
// the head at hoff[r] with the sampler's facts and cuts.
template <int kCap, int kT>
__global__ void __launch_bounds__(kT, kT == 128 ? 12 : (kCap <= 1024 ? HP_HEAD_SORT_MINB : 1)) k_head_sort(
    hp_query_layout L, const double* __restrict__ dirs, const double* __restrict__ slopes,
    const int64_t* __restrict__ off, const int* __restrict__ rays, const int64_t* __restrict__ soff,
    const int64_t* __restrict__ hoff,
    const RayMeta* __restrict__ meta, const unsigned* __restrict__ sc_key, const int* __restrict__ sc_slot,
    const uint4* __restrict__ sel, const int* __restrict__ list, const int* __restrict__ list_n, int whole,
    double* __restrict__ head_t, int* __restrict__ head_id, double* __restrict__ head_d, int* __restrict__ plen,
    int* __restrict__ facts, double* __restrict__ cut_t, double* __restrict__ cut_d, Params SP,
    float* __restrict__ head_u, unsigned long long* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char dyn[];
    HeadSmem<kCap>& F = *reinterpret_cast<HeadSmem<kCap>*>(dyn);
    const double4* __restrict__ rel4 = reinterpret_cast<const double4*>(L.rel4);
    const int tid = threadIdx.x;
    const int nr = *list_n;
    for (;;) {  // rays claimed dynamically (head lengths vary: no static tail)
        if (tid == 0) F.next = int(atomicAdd(work, 1ull));
        __syncthreads();
        const int k = F.next;
        if (k >= nr) break;
        const int64_t i = list[k], r = rays ? rays[i] : i;  // output i, ray r
        const int64_t so = soff[r];
        const int q = int(off[r + 1] - off[r]);
        const RayMeta M = meta[r];
        const bool all = q <= whole;
        unsigned kc = 0xffffffffu, kout = 0xffffffffu;
        int S = q;  // pairs to stage
        if (!all) {
            const uint4 sv = sel[i];
            kc = sv.x;
            S = int(sv.y);
            kout = sv.z;
        }
        HP_ASSERT(S <= kCap && S <= q);
        if (tid == 0) {
            F.cnt = F.keep = F.fcount = 0;
            F.fbad = M.bad;
            F.cut_d2 = ~0ull;
            F.kout = kout;
            F.thi = 0u;
        }
        // every slot in flight at once: a whole ray's from its match scratch, a
        // cut ray's selected ones from where k_head_select compacted them
        const int* src = all ? sc_slot + so : head_id + hoff[i];
        for (int e = tid; e < S; e += kT) cp_async4(&F.slot[e], src + e);
        cp_commit();
        for (int j = tid; j <= kCoarse; j += kT) F.chist[j] = 0;
        for (int j = tid; j <= S; j += kT) F.hist[j] = 0;
        cp_wait<0>();
        __syncthreads();
        // exact t / dist^2 / id of every staged pair; long rays keep t < T_c
        // (the trimmed pairs, t >= T_c, end up last in the order below)
        const double d0 = dirs[3 * r], d1 = dirs[3 * r + 1], d2v = dirs[3 * r + 2];
        const double Tc = (all || kc == 0xffffffffu) ? CUDART_INF : double(from_fkey(kc + 1u));
        // the rank's coarse map, counted in the same pass: [lower bound of every
        // t, T_c (cut rays) or the largest key (whole rays)]; a t above it lands
        // in the last bin (the map stays monotone: the order is unchanged)
        const float tlo = from_fkey(M.kmin);
        const float thi = all ? from_fkey(M.kmax) : float(Tc);
        const float cscale = coarse_scale(tlo, thi);
        const bool coarse = S > 64;  // rank_segment ranks up to 64 directly
        int nkeep = 0;
        for (int e = tid; e < S; e += kT) {
            const double4 a = rel4[F.slot[e]];
            const double t = cone_t(a.x, a.y, a.z, d0, d1, d2v);
            F.t[e] = t;
            F.d2[e] = cone_dist2(a.x, a.y, a.z, t, d0, d1, d2v);
            F.id[e] = int(__double_as_longlong(a.w));
            nkeep += t < Tc;
            if (coarse) {  // CTA-uniform
                const float x = coarse_of(t, tlo, cscale);
                F.bk[e] = __float_as_uint(x);  // over slot[e], read above by this thread
                const int b = min(int(x), kCoarse - 1);
                const unsigned peers = __match_any_sync(__activemask(), b);
                if (lane_id() == __ffs(peers) - 1) atomicAdd(&F.chist[b], __popc(peers));
            }
        }
        nkeep = warp_sum(nkeep);
        if (lane_id() == 0 && nkeep) atomicAdd(&F.keep, nkeep);
        __syncthreads();
        if (S > 0)
            rank_segment<kCap, kT, true>(S, tlo, thi, F.t, F.id, F.bk, F.hist, F.lst, F.perm, F.chist, F.scan_sh);
        const int Lh = F.keep;
        const int64_t ho = hoff[i];
        HP_ASSERT(Lh <= S && ho + Lh <= hoff[i + 1]);
        const double r0 = Lh > 0 ? dmul(__ldg(slopes + r), F.t[F.perm[0]]) : 0.0;
        int cnt = 0;
        bool bad = false;
        unsigned long long md = ~0ull;
        constexpr int kPer = kCap / kT;
        double tv[kPer], dv[kPer];  // this thread's head entries, for the bound factors below
#pragma unroll
        for (int c = 0; c < kPer; c++) {
            const int p = tid + c * kT;
            if (p >= S) break;
            const int e = F.perm[p];
            const double t = F.t[e], dd = F.d2[e];
            if (p < Lh) {
                const double d = sqrt(dd);
                tv[c] = t;
                dv[c] = d;
                head_t[ho + p] = t;
                head_id[ho + p] = F.id[e];
                head_d[ho + p] = d;
                cnt += d <= r0;
                bad |= !(fabs(t) <= DBL_MAX) || !(dd <= DBL_MAX);
            } else {
                md = min(md, dkey(dd));
            }
        }
        cnt = warp_sum(cnt);
        const bool anybad = __any_sync(0xffffffffu, bad);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) md = min(md, __shfl_xor_sync(0xffffffffu, md, o));
        if (lane_id() == 0) {
            if (cnt) atomicAdd(&F.fcount, cnt);
            if (anybad) atomicOr(&F.fbad, 1);
            if (md != ~0ull) atomicMin(&F.cut_d2, md);
        }
        __syncthreads();
        if (tid == 0) {
            plen[i] = Lh;
            facts[i] = (F.fbad || Lh == 0) ? -1 : F.fcount;
            // lower bounds of the left-out t / dist: a pair never staged has
            // t >= its key (> K_c) and an unknown dist (0); a trimmed pair's
            // are exact (the smallest trimmed t is the next in order)
            const bool unstaged = !all && F.kout != 0xffffffffu;
            double ct = CUDART_INF, cd = CUDART_INF;
            if (unstaged) {
                ct = double(from_fkey(F.kout));
                cd = 0.0;
            }
            if (Lh < S) {
                ct = fmin(ct, F.t[F.perm[Lh]]);
                cd = fmin(cd, sqrt(dkey_inv(F.cut_d2)));
            }
            cut_t[i] = ct;
            cut_d[i] = cd;
        }
        // The sampler's bound factors u_j >= fl(1 - alpha_j) for the head (the
        // plan's bound chain then only multiplies them): when every candidate
        // is eligible from the start (facts >= K, so j* = 0), u_j is
        // bound_factor_ring's (hp_sample_core.cuh) over the K candidates ending
        // at j, here from the sorted head in shared memory; rounded up to
        // float (still an upper bound); -1 where a member is not in j's pool.
        if (head_u && SP.K <= 32 && Lh >= SP.K && !F.fbad && F.fcount >= SP.K) {  // uniform in the CTA
            __syncthreads();  // F.t / F.d2 in element order are no longer read
#pragma unroll
            for (int c = 0; c < kPer; c++) {
                const int p = tid + c * kT;
                if (p < Lh) {
                    F.t[p] = tv[c];
                    F.d2[p] = dv[c];  // dist, in head order
                }
            }
            __syncthreads();
            const double slope = __ldg(slopes + r);
            const int nu = min(Lh, HP_HEAD_U_MAX);  // the chain rarely needs more; the plan computes the rest
            for (int p = tid; p < nu; p += kT) {
                const double tj = F.t[p], rj = dmul(slope, tj);
                const int i0 = p >= SP.K - 1 ? p - SP.K + 1 : 0;
                double sum = 0.0;
                bool ok = true;
                for (int k = 0; k < SP.K; k++) {
                    const double di = F.d2[i0 + k];
                    ok &= !(di > rj);
                    sum = dadd(sum, dadd(fabs(dsub(F.t[i0 + k], tj)), di));
                }
                head_u[ho + p] = ok ? __double2float_ru(factor_from_sum(sum, SP.K, SP)) : -1.0f;
            }
            for (int p = nu + tid; p < Lh; p += kT) head_u[ho + p] = -1.0f;  // the plan computes these
        } else if (head_u) {
            for (int p = tid; p < Lh; p += kT) head_u[ho + p] = -1.0f;
        }
        __syncthreads();
    }
}

struct HeadWs {
    void* scan;
    int64_t* soff;
    RayMeta* meta;
    int* lists;
    int* counts;
    uint4* sel;
    unsigned* key;
    int* slot;
    unsigned long long* work;  // work counters of the dynamically scheduled kernels
};

HeadWs carve_head(Carver& c, int64_t m, int64_t cap) {
    HeadWs w;
    const int64_t mm = m > 0 ? m : 1;
    w.scan = c.take<char>(scan_workspace_bytes(m + 1));
    w.soff = c.take<int64_t>(m + 1);
    w.meta = c.take<RayMeta>(mm);
    w.lists = c.take<int>(3 * mm);
    w.counts = c.take<int>(64);
    w.sel = c.take<uint4>(mm);
    w.key = c.take<unsigned>(cap > 0 ? cap : 1);
    w.slot = c.take<int>(cap > 0 ? cap : 1);
    w.work = c.take<unsigned long long>(4);  // [0] scan groups, [1] / [2] small / big sort rays
    return w;
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_head_workspace_bytes(int64_t m, int64_t capacity, size_t* bytes) {
    Carver c(nullptr, 0);
    carve_head(c, m, capacity);
    *bytes = c.used + 256;
    return HP_OK;
}

extern "C" int hp_head_count(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                             int64_t pad, const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                             const double* t_near, const double* t_far, const double* slopes, int64_t m,
                             int64_t* offsets, int64_t* head_off, int64_t* probes, int64_t* scanned,
                             int64_t capacity, void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(check_common(layout, pad, m, padded_w, padded_h));
    if (!layout.rel4 || !layout.relf || !head_off) {
        set_error("hp_head_count: the layout's relf / rel4 and head_off are required");
        return HP_EINVAL;
    }
    Carver cv(workspace, workspace_bytes);
    HeadWs w = carve_head(cv, m, capacity);
    if (!cv.ok()) {
        set_error("hp_head_count: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Rays R{pixels, pixel_stride, dirs, t_near, t_far, slopes};
    const QCam QC = make_qcam(cam);
    if (m > 0) {
        const int occ = kernel_occupancy((const void*)k_head_scan, kThreads, sizeof(HeadScanSmem));
        if (occ < 0) return occ;
        if (cudaMemsetAsync(w.work, 0, 4 * sizeof(unsigned long long), s) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "hp_head_count memset");
        TimedSpan ts("k_head_scan", s);
        k_head_scan<<<group_grid(m, occ), kThreads, sizeof(HeadScanSmem), s>>>(
            layout, padded_w, int(pad), R, QC, m, w.soff, w.key, w.slot, w.meta, offsets, head_off, probes, scanned,
            capacity, w.work);
        HP_CHECK_LAUNCH("k_head_scan");
    }
    HP_TRY(exclusive_scan_i64(offsets, offsets, m, w.scan, s));
    HP_TRY(exclusive_scan_i64(head_off, head_off, m, w.scan, s));
    if (m > 0) {
        k_mark_overflow<<<1, 1, 0, s>>>(reinterpret_cast<const int64_t*>(w.work + 3), capacity, offsets + m);
        HP_CHECK_LAUNCH("k_mark_overflow");
    }
    return HP_OK;
}

extern "C" int hp_head_sort(hp_query_layout layout, const double* dirs, const double* slopes, int64_t m,
                            const int64_t* offsets, const int32_t* rays, int64_t n, const int64_t* head_off,
                            int32_t want, int32_t whole, double* head_t, int32_t* head_ids, double* head_dist,
                            int32_t* plen, int32_t* facts, double* cut_t, double* cut_d,
                            const hp_sampler_params* sampler, float* head_u, int64_t capacity,
                            void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    // (the long-head mode needs a ray list: hp_head_count spaces head_off for 1024-entry heads)
    if (m < 0 || want < 1 || want > kHeadLong || whole < want || whole > kHeadLong || (rays && (n < 0 || n > m)) ||
        (!rays && whole > kHeadCap) ||
        (m > 0 && (!dirs || !slopes || !facts || !plen || !cut_t || !cut_d || !layout.rel4))) {
        set_error("hp_head_sort: invalid arguments (1 <= want <= whole <= %d with a ray list, else <= %d; n <= m)",
                  kHeadLong, kHeadCap);
        return HP_EINVAL;
    }
    // whole > kHeadCap: the long-head mode (heads up to 2048 in a <2048, 256> configuration, longer
    // ones in <4096, 512>)
    const bool lng = whole > kHeadCap;
    const int small = lng ? kHeadMid : kHeadSmall, cap = lng ? kHeadLong : kHeadCap;
    Carver cv(workspace, workspace_bytes);
    HeadWs w = carve_head(cv, m, capacity);
    if (!cv.ok()) {
        set_error("hp_head_sort: workspace too small");
        return HP_ESPACE;
    }
    const int64_t nout = rays ? n : m;  // outputs (rays[i] or i)
    if (nout == 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(w.counts, 0, 3 * sizeof(int), s) != cudaSuccess ||
        cudaMemsetAsync(w.work + 1, 0, 2 * sizeof(unsigned long long), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_head_sort memset");
    const int* list_small = w.lists;
    const int* list_big = w.lists + nout;
    const int* list_cut = w.lists + 2 * nout;
    k_head_classes<<<grid_for(nout, 256), 256, 0, s>>>(offsets, rays, nout, whole, small, w.lists, w.counts, plen,
                                                       facts, cut_t, cut_d, offsets + m);
    HP_CHECK_LAUNCH("k_head_classes");
    {
        constexpr auto kselect = k_head_select<kHeadCap>;
        const int occ_sel = kernel_occupancy((const void*)kselect, 128, 0);
        if (occ_sel < 0) return occ_sel;
        TimedSpan ts("k_head_select", s);
        kselect<<<device_sms() * occ_sel, 128, 0, s>>>(offsets, rays, w.soff, w.meta, want, whole, cap, small, w.key,
                                                       w.slot, head_off, head_ids, w.sel, list_cut, w.counts + 2,
                                                       w.lists, w.counts, nout);
        HP_CHECK_LAUNCH("k_head_select");
    }
    Params SP{};
    if (sampler && head_u) {
        SP.K = sampler->k_neighbors;
        SP.gamma = sampler->gamma;
        SP.beta2 = sampler->beta2;
        SP.inv_beta2_up = nextafter(1.0 / sampler->beta2, INFINITY);  // as hp_sample.cu to_params
        SP.inv_k_up = nextafter(1.0 / double(SP.K), INFINITY);
    } else {
        head_u = nullptr;
    }
    if (lng) {
        constexpr auto kmid = k_head_sort<kHeadMid, 256>;
        constexpr auto klong = k_head_sort<kHeadLong, 512>;
        const int occ_mid = kernel_occupancy((const void*)kmid, 256, sizeof(HeadSmem<kHeadMid>));
        if (occ_mid < 0) return occ_mid;
        const int occ_long = kernel_occupancy((const void*)klong, 512, sizeof(HeadSmem<kHeadLong>));
        if (occ_long < 0) return occ_long;
        TimedSpan ts("k_head_sort", s);
        kmid<<<device_sms() * occ_mid, 256, sizeof(HeadSmem<kHeadMid>), s>>>(
            layout, dirs, slopes, offsets, rays, w.soff, head_off, w.meta, w.key, w.slot, w.sel, list_small, w.counts,
            whole, head_t, head_ids, head_dist, plen, facts, cut_t, cut_d, SP, head_u, w.work + 1);
        HP_CHECK_LAUNCH("k_head_sort mid");
        klong<<<device_sms() * occ_long, 512, sizeof(HeadSmem<kHeadLong>), s>>>(
            layout, dirs, slopes, offsets, rays, w.soff, head_off, w.meta, w.key, w.slot, w.sel, list_big,
            w.counts + 1, whole, head_t, head_ids, head_dist, plen, facts, cut_t, cut_d, SP, head_u, w.work + 2);
        HP_CHECK_LAUNCH("k_head_sort long");
        return HP_OK;
    }
    constexpr auto ksmall = k_head_sort<kHeadSmall, 128>;
    constexpr auto kbig = k_head_sort<kHeadCap, 256>;
    const int occ_small = kernel_occupancy((const void*)ksmall, 128, sizeof(HeadSmem<kHeadSmall>));
    if (occ_small < 0) return occ_small;
    const int occ_big = kernel_occupancy((const void*)kbig, 256, sizeof(HeadSmem<kHeadCap>));
    if (occ_big < 0) return occ_big;
    TimedSpan ts("k_head_sort", s);
    ksmall<<<device_sms() * occ_small, 128, sizeof(HeadSmem<kHeadSmall>), s>>>(
        layout, dirs, slopes, offsets, rays, w.soff, head_off, w.meta, w.key, w.slot, w.sel, list_small, w.counts,
        whole, head_t, head_ids, head_dist, plen, facts, cut_t, cut_d, SP, head_u, w.work + 1);
    HP_CHECK_LAUNCH("k_head_sort small");
    kbig<<<device_sms() * occ_big, 256, sizeof(HeadSmem<kHeadCap>), s>>>(
        layout, dirs, slopes, offsets, rays, w.soff, head_off, w.meta, w.key, w.slot, w.sel, list_big,
        w.counts + 1, whole, head_t, head_ids, head_dist, plen, facts, cut_t, cut_d, SP, head_u, w.work + 2);
    HP_CHECK_LAUNCH("k_head_sort");
    return HP_OK;
}
