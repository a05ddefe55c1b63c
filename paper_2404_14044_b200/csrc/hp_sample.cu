// hp_sample.cu — adaptive primary-surface sampling over the query CSR.
//
// Reference: _kernels.sample_batch (_kernels.py:552-700); host wrapper
// sampler.sample_batch_arrays (sampler.py:196-217).
//
// Per ray (candidates already (t, id)-sorted by the query):
//   for each candidate j in order:
//     r_j = slope * t_j; pool = {i : ds_i <= r_j} if it has >= K members,
//     else all candidates; the K nearest by d2 = (t_i - t_j)^2 + ds_i^2
//     (ties: smaller i first); udf_j = mean of their sqrt(d2) (summed in
//     ascending order); alpha_j = gamma * exp(-(udf_j^2) / beta^2);
//     optional colour = inverse-distance blend of the selected points.
//   front to back: w_j = alpha_j * T, T *= 1 - alpha_j; t_end = T.
//   retention: eps mode keeps w_j >= eps; tau mode keeps the prefix while
//   T (before j) >= tau_min.
//
// Kernels (hp_sample_run / hp_sample_emit):
//   k_sample_plan    warp per ray: fast-path preconditions (or the query's
//                    facts), j*, and a monotone upper bound of the reference's
//                    transmittance (bound factors from window members, a
//                    shared-memory ring of the last 64 candidates) -> the
//                    exact region [0, E): E = je, the index where retention is
//                    decided, when the product is proved to reach exactly 0
//                    (or in exit mode), else q
//   k_sample_expand  exact slot -> ray
//   k_sample_exact   thread per exact candidate: K nearest, udf, alpha, colour
//   k_sample_retain  warp per ray: the reference's sequential compositing
//                    over [0, E), retention (compacted in place), t_end
//   k_emit           retained candidates -> the output CSR
// Exact reformulations:
//   * use_el(j) = (#{ds_i <= r_j} >= K) = (ds_(K) <= r_j) is monotone in j
//     when t is sorted and slope >= 0: a search over j finds the first j
//     where it holds.
//   * the exact K-nearest search expands outward from j in t order and stops
//     when (t_edge - t_j)^2 > the K-th best d2; selection key (d2, i)
//     reproduces the reference's strict-< insertion.
//   * only candidates before the retention decision need the exact alpha;
//     the bound locates that point and, in exact-t_end mode, proves when the
//     reference's product underflows to exactly 0.
// Rays violating the preconditions (unsorted t, negative/NaN values) take the
// reference's direct loops, still on the device.
#include <math_constants.h>

#include <cfloat>
#include <climits>
#include <cmath>

#include "hp_common.cuh"
#include "hp_sample_core.cuh"

namespace hp {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef HP_PLAN_CPASYNC
#define HP_PLAN_CPASYNC 1
#endif
#ifndef HP_PLAN_F32
#define HP_PLAN_F32 1  // fp32 ring bound factors in k_sample_plan
#endif
#ifndef HP_PLAN_CLAIM
#define HP_PLAN_CLAIM 4  // rays per warp claim in k_sample_plan
#endif
#ifndef HP_PLAN_AHEAD
#define HP_PLAN_AHEAD 2  // chunks in flight
#endif
// plan ring: the last 64 candidates (bound factors, K <= 32) + the chunks in
// flight with cp.async
constexpr int kRing = HP_PLAN_CPASYNC ? (HP_PLAN_AHEAD <= 2 ? 128 : 256) : 64;

// Path counters: rays, fast rays, proved-zero rays, exact evaluations,
// candidates, bound evaluations.  Read with hp_sample_debug_counters().
// Compiled in with -DHP_DEBUG_COUNTERS only: same-address global atomics per
// ray serialise in L2 and cost ~0.5 ms per cfg2 frame.
__device__ unsigned long long g_dbg[8];
#ifdef HP_DEBUG_COUNTERS
#define HP_DBG_ADD(k, v) atomicAdd(&g_dbg[k], (unsigned long long)(v))
#else
#define HP_DBG_ADD(k, v) ((void)0)
#endif


struct Csr {
    const int64_t* off;
    const int64_t* ids;
    const double* t;
    const double* ds;
    const double* slopes;
    const double* colors;
    int64_t m;
    const int32_t* facts;  // optional per-ray facts from hp_query_fill (NULL: compute)
    // prefix mode (hp_query_prefix; start == NULL: CSR mode).  Ray r's
    // candidates are the first len[r] of its off[r+1] - off[r] matches, at
    // start[r]; the rest all have t >= cut_t[r] and dist >= cut_d[r].
    const int64_t* start;
    const int32_t* len;
    const int32_t* ids32;
    const double* cut_t;
    const double* cut_d;
    int32_t* flag;  // [m + 1]: 1 = the ray needs its full CSR; flag[m] = count
    const float* head_u;  // optional precomputed bound factors (hp_head_sort), at start[r]
    __device__ __forceinline__ int64_t lo(int64_t r) const { return start ? start[r] : off[r]; }
    __device__ __forceinline__ int n(int64_t r) const { return start ? len[r] : int(off[r + 1] - off[r]); }
    __device__ __forceinline__ int qtrue(int64_t r) const { return int(off[r + 1] - off[r]); }
    __device__ __forceinline__ int64_t id(int64_t k) const { return ids32 ? int64_t(ids32[k]) : ids[k]; }
};

struct Outputs {
    int64_t* r_id;
    double *r_t, *r_dist, *r_udf, *r_alpha, *r_w, *r_color;
    int64_t* r_knn_id;  // [R, K] with P.emit_knn
    double* r_knn_w;
};

struct RayOut {  // per-ray results of pass 1
    int64_t* rcount;  // retained count (scanned into r_off)
    double* t_end;
};

// ---- plan (k_sample_plan): one warp per ray, no shared memory.
// Fast-path preconditions, j* (first j where use_el holds), and the bound
// chain: je (retention is decided before je) and whether the reference's
// transmittance provably underflows to exactly 0.  plan[ray] =
// (jstar, je, flags: 1 fast | 2 proved_zero, q).
__device__ void plan_ray(const Csr& C, const Params& P, int64_t ray, int4* __restrict__ plan,
                         int64_t* __restrict__ ecnt, double* __restrict__ rt, double* __restrict__ rd, float2* rf) {
    const int lane = lane_id();
    const int64_t lo = C.lo(ray);
    const int q = C.n(ray);  // candidates present (prefix mode: the prefix)
    const int qt = C.start ? C.qtrue(ray) : q;
    const bool partial = q < qt;
    const int fact = C.facts ? C.facts[ray] : -1;
    // prefix mode: a ray whose work may reach past its prefix is flagged for
    // the full path (no facts, or a prefix shorter than K)
    // flag values say why (diagnostics; any nonzero value means "flagged"):
    // 1 no facts / head shorter than K, 2 preconditions, 3 eligibility past
    // the head, 4 retention / the zero proof past the head, 5 K nearest past it
    auto flag_out = [&](int why) {
        if (lane == 0) {
            plan[ray] = make_int4(0, 0, 0, 0);
            ecnt[ray] = 0;
            C.flag[ray] = why;
        }
    };
    if (partial && (fact < 0 || q < P.K)) return flag_out(1);
    if (C.start && lane == 0) C.flag[ray] = 0;
    if (q == 0) {
        if (lane == 0) {
            plan[ray] = make_int4(0, 0, 0, 0);
            ecnt[ray] = 0;
        }
        return;
    }
    const double slope = C.slopes[ray];
    const double* T = C.t + lo;
    const double* DS = C.ds + lo;
    const double thr = P.eps_mode ? P.eps : P.tau_min;
    const RayView V{T, DS};

    // fast-path preconditions + count of candidates within r_0 (use_el holds
    // from j = 0 when it reaches K, the common case on dense surfaces)
    bool ok = slope >= 0.0 && slope <= DBL_MAX;
    int c0cnt = 0;
    if (fact >= 0) {  // the query's sort established the preconditions
        c0cnt = lane == 0 ? fact : 0;
    } else {
        const double r0 = dmul(slope, ldg(T));
#pragma unroll 4
        for (int k = lane; k < q; k += 32) {
            const double tk = ldg(T + k), dk = ldg(DS + k);
            ok &= (fabs(tk) <= DBL_MAX) && (dk >= 0.0) && (dk <= DBL_MAX);
            if (k + 1 < q) ok &= !(ldg(T + k + 1) < tk);
            c0cnt += (dk <= r0);
        }
    }
    const bool fast = __all_sync(0xffffffffu, ok);
    if (partial && !fast) return flag_out(2);
    int jstar = 0;
    if (fast) {
        if (warp_sum(c0cnt) >= P.K) {
            jstar = 0;
        } else if (qt < P.K) {
            jstar = q;
        } else {
            // first j with #{ds_i <= slope * t_j} >= K (monotone in j)
            jstar = warp_first_true(q, [&](int j) {
                const double rj = dmul(slope, V.t(j));
                int c = 0;
                for (int i = 0; i < q; i++) c += (V.d(i) <= rj);
                return c >= P.K;
            });
            // prefix counts are the full counts while r_j < cut_d (the
            // left-out matches are all farther out); beyond, unknown
            if (partial && jstar > 0 && !(dmul(slope, V.t(jstar - 1)) < __ldg(C.cut_d + ray))) return flag_out(3);
        }
    }
    // ---- 1. bound chain (fast path): chain_chunk over 32 candidates at a time
    int je = q;  // retention is decided before je
    bool proved_zero = false;
    unsigned long long nbound = 0;
    if (fast) {
        Chain S;
        S.je = q;
        double tb = 0.0;  // the ray's base t for the fp32 bound terms
#if HP_PLAN_CPASYNC
        // the ring is filled by cp.async two chunks ahead (no registers held
        // across the chunk; the chunk's own work does not cover a DRAM trip)
        auto fetch = [&](int c) {
            const int jj = c + lane;
            if (P.K <= 32 && jj < q) {
                cp_async8(&rt[jj & (kRing - 1)], T + jj);
                cp_async8(&rd[jj & (kRing - 1)], DS + jj);
            }
            cp_commit();
        };
        if (!(C.head_u && jstar == 0 && P.K <= 32)) {
#pragma unroll
            for (int a = 0; a < HP_PLAN_AHEAD; a++) fetch(32 * a);
        }
#else
        // this lane's (t, ds) of the current chunk, loaded one chunk ahead
        double tn = lane < q ? ldg(T + lane) : 0.0, dn = lane < q ? ldg(DS + lane) : 0.0;
#endif
        // precomputed factors (hp_head_sort) when every candidate is eligible
        const float* HU = (C.head_u && jstar == 0 && P.K <= 32) ? C.head_u + lo : nullptr;
        float hu_next = (HU && lane < q) ? __ldg(HU + lane) : 1.0f;  // one chunk ahead
        for (int c0 = 0; c0 < q; c0 += 32) {
            const int j = c0 + lane;
            double u = 1.0;
            if (HU) {
                const float hu = hu_next;
                hu_next = j + 32 < q ? __ldg(HU + j + 32) : 1.0f;
                if (j < q) {
                    u = double(hu);
                    if (u < 0.0) u = bound_factor(V, q, j, jstar, slope, P);
                }
            } else if (P.K <= 32) {
#if HP_PLAN_CPASYNC
                cp_wait<HP_PLAN_AHEAD - 1>();  // chunk c0 has landed
                __syncwarp();
                const double tj = j < q ? rt[j & (kRing - 1)] : 0.0;
                float thi = 0.0f, rj_lo = 0.0f;
                if (P.f32_bounds) {
                    if (c0 == 0) tb = __shfl_sync(0xffffffffu, tj, 0);
                    const double dj = j < q ? rd[j & (kRing - 1)] : 0.0;
                    rf[j & (kRing - 1)] = make_float2(__double2float_rd(__dsub_rd(tj, tb)), __double2float_ru(dj));
                    thi = __double2float_ru(__dsub_ru(tj, tb));
                    rj_lo = __double2float_rd(__dmul_rd(slope, tj));
                    __syncwarp();
                }
                fetch(c0 + 32 * HP_PLAN_AHEAD);  // its slots are outside the windows still to be read
#else
                const double tj = tn, dj = dn;
                const int jn = j + 32;
                tn = jn < q ? ldg(T + jn) : 0.0;
                dn = jn < q ? ldg(DS + jn) : 0.0;
                __syncwarp();
                rt[j & (kRing - 1)] = tj;
                rd[j & (kRing - 1)] = dj;
                __syncwarp();
#endif
                if (j < q) {
                    const bool use_el = j >= jstar;
                    const int ksel = use_el ? P.K : (q < P.K ? q : P.K);
#if HP_PLAN_CPASYNC
                    if (P.f32_bounds && j >= ksel - 1)
                        u = bound_factor_ringf<kRing>(rf, j, thi, rj_lo, ksel, use_el, P);
                    else
#endif
                    u = (j >= P.K - 1 || c0 + 32 >= min(q, P.K))
                            ? bound_factor_ring<kRing>(rt, rd, q, j, tj, jstar, slope, P)
                            : -1.0;
                    if (u < 0.0) u = bound_factor(V, q, j, jstar, slope, P);
                }
            } else if (j < q) {
                u = bound_factor(V, q, j, jstar, slope, P);
            }
            nbound += 32;
            if (chain_chunk(S, u, c0, min(32, q - c0), q, thr, P)) break;
        }
#if HP_PLAN_CPASYNC
        cp_wait<0>();  // nothing may land in the ring once the next ray uses it
        __syncwarp();
#endif
        je = S.je;
        proved_zero = S.proved_zero;
    }
    // prefix mode: retention (and, exact t_end, the zero) must be decided
    // inside the prefix
    if (partial && (je == q || (P.exact_t_end && !proved_zero))) return flag_out(4);
    if (lane == 0) {
        plan[ray] = make_int4(jstar, je, (fast ? 1 : 0) | (proved_zero ? 2 : 0), q);
        // exact region [0, E): everything unless retention is decided before je
        // and (exact t_end) the transmittance is proved to reach exactly 0
        ecnt[ray] = (!fast || (P.exact_t_end && !proved_zero)) ? q : je;
        HP_DBG_ADD(5, nbound);
    }
}

__global__ void __launch_bounds__(kThreads) k_sample_plan(Csr C, Params P, int4* __restrict__ plan,
                                                          int64_t* __restrict__ ecnt,
                                                          unsigned long long* __restrict__ work) {
    __shared__ double ring[kWarps][2][kRing];  // recent candidates' t / ds per warp
    __shared__ float2 ringf[kWarps][kRing];    // their fp32 bound terms
    WarpClaim<HP_PLAN_CLAIM> claim(work);  // chain lengths vary widely: rays claimed dynamically
    int64_t ray;
    while (claim.next(C.m, ray))
        plan_ray(C, P, ray, plan, ecnt, ring[warp_id()][0], ring[warp_id()][1], ringf[warp_id()]);
}

// r_off[m] = -(exact slots needed) when the caller's capacity is short
__global__ void k_mark_exact_overflow(const int64_t* __restrict__ need_at, int64_t cap, int64_t* __restrict__ total) {
    if (*need_at > cap) *total = -*need_at;
}

// candidate slot -> ray: a warp per 32 consecutive rays, whose slots are one
// contiguous range [eoff[r0], eoff[r0 + 32]); lane l fills slots l, l + 32,
// ... of it (coalesced), the ray found by a binary search over the lanes'
// inclusive counts
__global__ void k_sample_expand(int64_t m, const int64_t* __restrict__ eoff, int* __restrict__ cand_ray, int64_t cap) {
    if (eoff[m] > cap) return;  // exact scratch too small (hp_sample_run reports it in r_off[m])
    const int lane = lane_id();
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r0 = (blockIdx.x * int64_t(blockDim.x >> 5) + warp_id()) * 32; r0 < m; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        const int n = r < m ? int(eoff[r + 1] - eoff[r]) : 0;
        const int64_t base = __shfl_sync(0xffffffffu, eoff[r0], 0);
        const int incl = warp_incl_scan(n);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int b0 = 0; b0 < total; b0 += 32) {  // whole warp in every round (shuffles)
            const int sidx = b0 + lane;
            int owner = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= sidx) owner += step;
            }
            if (sidx < total) {
                HP_ASSERT(base + sidx < cap);
                cand_ray[base + sidx] = int(r0 + owner);
            }
        }
    }
}

// Per exact candidate, flat over all rays (ray r owns slots [eoff[r],
// eoff[r+1])).  After k_sample_retain the first rcount[r] slots of each ray
// hold its retained candidates, compacted in place: ray[] then holds the
// candidate's index j within the ray and w[] its weight.
struct Exact {
    double* udf;
    double* alpha;
    double* w;
    double* col;      // [n, 3]
    int64_t* knn_id;  // [n, K] with P.emit_knn
    double* knn_w;
    int* ray;
    int64_t cap;
};

// One thread per exact candidate (all lanes busy regardless of how few
// candidates a ray needs): exact udf / alpha / colour of candidate j of ray.
template <class BestT, bool kKnn>
// HP_EXACT_MINB > 0: minimum resident CTAs per SM for the K <= 8 instances
// (an explicit 1 is not the same as none: ptxas then allots more registers)
#ifndef HP_EXACT_DYN
#define HP_EXACT_DYN 1  // k_sample_exact: candidates claimed 32 at a time per warp
#endif
#ifndef HP_EXACT_MINB
#define HP_EXACT_MINB 4
#endif
#if HP_EXACT_MINB > 0
#define HP_EXACT_BOUNDS __launch_bounds__(kThreads, BestT::kMax <= 8 ? HP_EXACT_MINB : 1)
#else
#define HP_EXACT_BOUNDS __launch_bounds__(kThreads)
#endif
__global__ void HP_EXACT_BOUNDS k_sample_exact(Csr C, Params P, const int4* __restrict__ plan,
                                                           const int64_t* __restrict__ eoff, Exact X,
                                                           unsigned long long* __restrict__ claim) {
    const int64_t n = eoff[C.m];
    if (n > X.cap) return;
    unsigned long long evals = 0;
#if HP_EXACT_DYN
    // 32 candidates per warp claimed dynamically (their costs vary widely:
    // a static stride leaves a tail)
    for (;;) {
        unsigned long long b = 0;
        if (lane_id() == 0) b = atomicAdd(claim, 32ull);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (int64_t(b) >= n) break;
        const int64_t c = int64_t(b) + lane_id();
        if (c >= n) continue;
#else
    (void)claim;
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n; c += int64_t(gridDim.x) * blockDim.x) {
#endif
        const int ray = X.ray[c];
        const int j = int(c - eoff[ray]);
        const int4 pl = plan[ray];
        const int64_t lo = C.lo(ray);
        const int q = pl.w;
        const RayView V{C.t + lo, C.ds + lo};
        double u, a, col[3] = {0.0, 0.0, 0.0};
        bool ok = true;
        if (C.start) {
            const int qt = C.qtrue(ray);
            ok = eval_exact<BestT>(V, q, qt, q < qt ? __ldg(C.cut_t + ray) : CUDART_INF, j, pl.z & 1, pl.x,
                                   C.slopes[ray], P, C.ids32 + lo, C.colors, u, a, col, evals,
                                   kKnn ? X.knn_id + c * P.K : nullptr, kKnn ? X.knn_w + c * P.K : nullptr);
        } else {
            eval_exact<BestT>(V, q, q, CUDART_INF, j, pl.z & 1, pl.x, C.slopes[ray], P, C.ids + lo, C.colors, u, a,
                              col, evals, kKnn ? X.knn_id + c * P.K : nullptr, kKnn ? X.knn_w + c * P.K : nullptr);
        }
        if (!ok) C.flag[ray] = 5;
        X.udf[c] = u;
        X.alpha[c] = a;
        if (P.want_color) {
            X.col[3 * c] = col[0];
            X.col[3 * c + 1] = col[1];
            X.col[3 * c + 2] = col[2];
        }
    }
#ifdef HP_DEBUG_COUNTERS
    evals = warp_sum(evals);
    if (lane_id() == 0 && evals) HP_DBG_ADD(3, evals);
#endif
}

// One warp per ray: the reference's sequential compositing over the exact
// region (_kernels.py:661-697), retention, transmittance.  Retained
// candidates are compacted to the front of the ray's exact slots (a retained
// candidate's position never exceeds its index, and every lane reads its
// chunk before any lane writes).
template <bool kKnn>
__device__ void retain_ray(const Csr& C, const Params& P, int64_t ray, const RayOut& RO,
                           const int4* __restrict__ plan, const int64_t* __restrict__ eoff, const Exact& X) {
    const int lane = lane_id();
    const int4 pl = plan[ray];
    const int q = pl.w;
    if (C.start && C.flag[ray]) {  // left to the full path
        if (lane == 0) {
            RO.rcount[ray] = 0;
            RO.t_end[ray] = CUDART_NAN;
            atomicAdd(C.flag + C.m, 1);
        }
        return;
    }
    if (q == 0) {
        if (lane == 0) {
            RO.rcount[ray] = 0;
            RO.t_end[ray] = 1.0;
        }
        return;
    }
    const bool fast = pl.z & 1, proved_zero = (pl.z >> 1) & 1;
    const double thr = P.eps_mode ? P.eps : P.tau_min;
    const int64_t e0 = eoff[ray];
    const int E = int(eoff[ray + 1] - e0);
    double Tr = 1.0, exit_T = -1.0;
    int nret = 0;
    for (int c0 = 0; c0 < E; c0 += 32) {
        const int j = c0 + lane;
        const double a = j < E ? X.alpha[e0 + j] : 0.0;
        const int n = min(32, E - c0);
        double wmine = 0.0;
        unsigned keep = 0;
        bool stop = false;
        for (int k = 0; k < n; k++) {
            if (!P.exact_t_end && Tr < thr) {  // exit mode: retention decided
                exit_T = Tr;
                stop = true;
                break;
            }
            const double ak = __shfl_sync(0xffffffffu, a, k);
            const double w = dmul(ak, Tr);
            const bool kp = P.eps_mode ? (w >= P.eps) : !(Tr < P.tau_min);
            if (kp) keep |= 1u << k;
            if (lane == k) wmine = w;
            Tr = dmul(Tr, dsub(1.0, ak));
        }
        if (keep) {
            const bool mine = (keep >> lane) & 1u;
            const int64_t dst = e0 + nret + __popc(keep & ((1u << lane) - 1));
            HP_ASSERT(!mine || (dst < e0 + E && dst <= e0 + j));
            double u = 0.0, c[3] = {0.0, 0.0, 0.0};
            if (mine) {
                u = X.udf[e0 + j];
                if (P.want_color)
                    for (int x = 0; x < 3; x++) c[x] = X.col[3 * (e0 + j) + x];
            }
            __syncwarp();
            if (mine) {
                X.udf[dst] = u;
                X.alpha[dst] = a;
                X.w[dst] = wmine;
                X.ray[dst] = j;
                if (P.want_color)
                    for (int x = 0; x < 3; x++) X.col[3 * dst + x] = c[x];
            }
            __syncwarp();
            if (kKnn) {  // the neighbour rows, 8 columns at a time (every read before any write)
                for (int b0 = 0; b0 < P.K; b0 += 8) {
                    int64_t kid[8];
                    double kw[8];
#pragma unroll
                    for (int b = 0; b < 8; b++)
                        if (mine && b0 + b < P.K) {
                            kid[b] = X.knn_id[(e0 + j) * P.K + b0 + b];
                            kw[b] = X.knn_w[(e0 + j) * P.K + b0 + b];
                        }
                    __syncwarp();
#pragma unroll
                    for (int b = 0; b < 8; b++)
                        if (mine && b0 + b < P.K) {
                            X.knn_id[dst * P.K + b0 + b] = kid[b];
                            X.knn_w[dst * P.K + b0 + b] = kw[b];
                        }
                    __syncwarp();
                }
            }
        }
        nret += __popc(keep);
        if (stop) break;
    }
    if (lane == 0) {
        HP_DBG_ADD(0, 1);
        HP_DBG_ADD(1, fast ? 1 : 0);
        HP_DBG_ADD(2, proved_zero ? 1 : 0);
        HP_DBG_ADD(4, q);
        double te;
        if (P.exact_t_end)
            te = (fast && proved_zero) ? 0.0 : Tr;
        else
            te = exit_T >= 0.0 ? exit_T : Tr;
        RO.rcount[ray] = nret;
        RO.t_end[ray] = te;
    }
}

template <bool kKnn>
__global__ void __launch_bounds__(kThreads) k_sample_retain(Csr C, Params P, RayOut RO, const int4* __restrict__ plan,
                                                            const int64_t* __restrict__ eoff, Exact X) {
    if (eoff[C.m] > X.cap) return;
    const int64_t warps = int64_t(gridDim.x) * kWarps;
    for (int64_t ray = int64_t(blockIdx.x) * kWarps + warp_id(); ray < C.m; ray += warps)
        retain_ray<kKnn>(C, P, ray, RO, plan, eoff, X);
}

#ifndef HP_EMIT_FLAT
#define HP_EMIT_FLAT 1  // k_emit: a warp per 32 consecutive rays, coalesced writes
#endif
#ifndef HP_RETAIN_SHORT
#define HP_RETAIN_SHORT 16  // rays of at most this many exact candidates: one thread each
#endif
// One thread per ray for the (common) rays with few exact candidates: the
// same sequential compositing as retain_ray, every read of a candidate
// before its (lower or equal) compacted slot is written; longer rays are
// listed for the warp-per-ray kernel below.
template <bool kKnn>
__global__ void __launch_bounds__(kThreads) k_sample_retain_short(Csr C, Params P, RayOut RO,
                                                                  const int4* __restrict__ plan,
                                                                  const int64_t* __restrict__ eoff, Exact X,
                                                                  int* __restrict__ longs,
                                                                  unsigned long long* __restrict__ nlong) {
    if (eoff[C.m] > X.cap) return;
    for (int64_t ray = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; ray < C.m;
         ray += int64_t(gridDim.x) * blockDim.x) {
        const int4 pl = plan[ray];
        const int q = pl.w;
        if (C.start && C.flag[ray]) {  // left to the full path
            RO.rcount[ray] = 0;
            RO.t_end[ray] = CUDART_NAN;
            atomicAdd(C.flag + C.m, 1);
            continue;
        }
        if (q == 0) {
            RO.rcount[ray] = 0;
            RO.t_end[ray] = 1.0;
            continue;
        }
        const int64_t e0 = eoff[ray];
        const int E = int(eoff[ray + 1] - e0);
        if (E > HP_RETAIN_SHORT) {
            longs[atomicAdd(nlong, 1ull)] = int(ray);
            continue;
        }
        const bool fast = pl.z & 1, proved_zero = (pl.z >> 1) & 1;
        const double thr = P.eps_mode ? P.eps : P.tau_min;
        double Tr = 1.0, exit_T = -1.0;
        int nret = 0;
        for (int j = 0; j < E; j++) {
            if (!P.exact_t_end && Tr < thr) {  // exit mode: retention decided
                exit_T = Tr;
                break;
            }
            const double a = X.alpha[e0 + j];
            const double w = dmul(a, Tr);
            if (P.eps_mode ? (w >= P.eps) : !(Tr < P.tau_min)) {
                const int64_t src = e0 + j, dst = e0 + nret;
                X.udf[dst] = X.udf[src];
                X.alpha[dst] = a;
                X.w[dst] = w;
                X.ray[dst] = j;
                if (P.want_color)
                    for (int x = 0; x < 3; x++) X.col[3 * dst + x] = X.col[3 * src + x];
                if (kKnn)
                    for (int b = 0; b < P.K; b++) {
                        X.knn_id[dst * P.K + b] = X.knn_id[src * P.K + b];
                        X.knn_w[dst * P.K + b] = X.knn_w[src * P.K + b];
                    }
                nret++;
            }
            Tr = dmul(Tr, dsub(1.0, a));
        }
        HP_DBG_ADD(0, 1);
        HP_DBG_ADD(1, fast ? 1 : 0);
        HP_DBG_ADD(2, proved_zero ? 1 : 0);
        HP_DBG_ADD(4, q);
        double te;
        if (P.exact_t_end)
            te = (fast && proved_zero) ? 0.0 : Tr;
        else
            te = exit_T >= 0.0 ? exit_T : Tr;
        RO.rcount[ray] = nret;
        RO.t_end[ray] = te;
    }
}

template <bool kKnn>
__global__ void __launch_bounds__(kThreads) k_sample_retain_long(Csr C, Params P, RayOut RO,
                                                                 const int4* __restrict__ plan,
                                                                 const int64_t* __restrict__ eoff, Exact X,
                                                                 const int* __restrict__ longs,
                                                                 const unsigned long long* __restrict__ nlong) {
    if (eoff[C.m] > X.cap) return;
    const int64_t n = int64_t(*nlong);
    const int64_t warps = int64_t(gridDim.x) * kWarps;
    for (int64_t k = int64_t(blockIdx.x) * kWarps + warp_id(); k < n; k += warps)
        retain_ray<kKnn>(C, P, longs[k], RO, plan, eoff, X);
}

// Copy the compacted retained candidates to the outputs (ray order).
template <bool kKnn>
__global__ void k_emit(Csr C, Params P, const int64_t* __restrict__ r_off, const int64_t* __restrict__ eoff,
                       Exact X, Outputs O) {
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + warp_id(); r < C.m; r += warps) {
        const int64_t o = r_off[r], n = r_off[r + 1] - o;
        if (n == 0) continue;
        const int64_t lo = C.lo(r), st = eoff[r];
        for (int64_t k = lane_id(); k < n; k += 32) {
            const int64_t j = lo + X.ray[st + k];
            O.r_id[o + k] = C.id(j);
            O.r_t[o + k] = C.t[j];
            O.r_dist[o + k] = C.ds[j];
            O.r_udf[o + k] = X.udf[st + k];
            O.r_alpha[o + k] = X.alpha[st + k];
            O.r_w[o + k] = X.w[st + k];
            if (P.want_color) {
                O.r_color[3 * (o + k)] = X.col[3 * (st + k)];
                O.r_color[3 * (o + k) + 1] = X.col[3 * (st + k) + 1];
                O.r_color[3 * (o + k) + 2] = X.col[3 * (st + k) + 2];
            }
            if (kKnn)
                for (int b = 0; b < P.K; b++) {
                    O.r_knn_id[(o + k) * P.K + b] = X.knn_id[(st + k) * P.K + b];
                    O.r_knn_w[(o + k) * P.K + b] = X.knn_w[(st + k) * P.K + b];
                }
        }
    }
}

// The same copy with a warp per 32 consecutive rays: their retained samples
// are one contiguous output range, so lane l writes samples l, l + 32, ...
// of it (coalesced); each sample's ray is found among the warp's 32 by a
// binary search over the inclusive counts held in the lanes.
template <bool kKnn>
__global__ void k_emit_flat(Csr C, Params P, const int64_t* __restrict__ r_off, const int64_t* __restrict__ eoff,
                            Exact X, Outputs O) {
    const int lane = lane_id();
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r0 = (blockIdx.x * int64_t(blockDim.x >> 5) + warp_id()) * 32; r0 < C.m; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        int n = 0;
        int64_t st = 0, lo = 0;
        if (r < C.m) {
            n = int(r_off[r + 1] - r_off[r]);
            if (n) {
                st = eoff[r];
                lo = C.lo(r);
            }
        }
        const int64_t o0 = __shfl_sync(0xffffffffu, r < C.m ? r_off[r] : 0, 0);
        const int incl = warp_incl_scan(n);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int base = 0; base < total; base += 32) {  // whole warp in every round (shuffles)
            const int sidx = base + lane;
            int owner = 0;  // first lane whose inclusive count exceeds sidx
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= sidx) owner += step;
            }
            const int excl = __shfl_sync(0xffffffffu, incl - n, owner);
            const int64_t sto = __shfl_sync(0xffffffffu, st, owner), loo = __shfl_sync(0xffffffffu, lo, owner);
            if (sidx >= total) continue;
            const int64_t k = sidx - excl, o = o0 + sidx;
            const int64_t j = loo + X.ray[sto + k];
            O.r_id[o] = C.id(j);
            O.r_t[o] = C.t[j];
            O.r_dist[o] = C.ds[j];
            O.r_udf[o] = X.udf[sto + k];
            O.r_alpha[o] = X.alpha[sto + k];
            O.r_w[o] = X.w[sto + k];
            if (P.want_color) {
                O.r_color[3 * o] = X.col[3 * (sto + k)];
                O.r_color[3 * o + 1] = X.col[3 * (sto + k) + 1];
                O.r_color[3 * o + 2] = X.col[3 * (sto + k) + 2];
            }
            if (kKnn)
                for (int b = 0; b < P.K; b++) {
                    O.r_knn_id[o * P.K + b] = X.knn_id[(sto + k) * P.K + b];
                    O.r_knn_w[o * P.K + b] = X.knn_w[(sto + k) * P.K + b];
                }
        }
    }
}

__global__ void k_primary(const int64_t* __restrict__ r_off, int64_t m, const int64_t* __restrict__ r_id,
                          const double* __restrict__ r_t, int64_t* __restrict__ pid, double* __restrict__ pt) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t a = r_off[r], b = r_off[r + 1];
        pid[r] = b > a ? r_id[a] : -1;
        if (pt) pt[r] = b > a ? r_t[a] : CUDART_NAN;
    }
}

__global__ void k_csr_stats(const int64_t* __restrict__ off, int64_t m, int64_t* __restrict__ out2) {
    int64_t mx = 0;
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t q = off[r + 1] - off[r];
        mx = q > mx ? q : mx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx ? v : mx;
    }
    if (lane_id() == 0 && mx > 0) atomicMax(reinterpret_cast<unsigned long long*>(out2 + 1), (unsigned long long)mx);
    if (blockIdx.x == 0 && threadIdx.x == 0) out2[0] = off[m];
}

struct SampleWs {
    int4* plan;
    int64_t* eoff;  // [m + 1] exact-candidate offsets
    Exact x;
    void* scan;
    unsigned long long* work;  // k_sample_plan's ray counter
    int* longs;                // rays left to the warp-per-ray retain
};

SampleWs carve_sample(Carver& c, int64_t m, int64_t xcap, bool color, int knn_k = 0) {
    SampleWs w;
    w.plan = c.take<int4>(m > 0 ? m : 1);
    w.eoff = c.take<int64_t>(m + 1);
    const int64_t xc = xcap > 0 ? xcap : 1;
    w.x.cap = xcap;
    w.x.udf = c.take<double>(xc);
    w.x.alpha = c.take<double>(xc);
    w.x.w = c.take<double>(xc);
    w.x.col = color ? c.take<double>(3 * xc) : nullptr;
    w.x.knn_id = knn_k > 0 ? c.take<int64_t>(xc * knn_k) : nullptr;
    w.x.knn_w = knn_k > 0 ? c.take<double>(xc * knn_k) : nullptr;
    w.x.ray = c.take<int>(xc);
    w.scan = c.take<char>(scan_workspace_bytes(m + 1));
    w.work = c.take<unsigned long long>(3);  // [0] k_sample_plan's rays, [1] the retain's long rays, [2] exact claims
    w.longs = c.take<int>(m > 0 ? m : 1);
    return w;
}

Params to_params(const hp_sampler_params* p) {
    Params P;
    P.K = p->k_neighbors;
    P.eps_mode = p->eps_mode;
    P.want_color = p->want_color;
    P.exact_t_end = p->exact_t_end;
    P.emit_knn = p->emit_knn;
    P.beta2 = p->beta2;
    P.gamma = p->gamma;
    P.eps = p->eps;
    P.tau_min = p->tau_min;
    // 1/beta2 rounded toward +inf on the host (fesetround-free): next double up
    const double r = 1.0 / p->beta2;
    P.inv_beta2_up = nextafter(r, INFINITY);
    P.inv_k_up = nextafter(1.0 / double(P.K), INFINITY);
    auto f_up = [](double x) {
        float f = float(x);
        return double(f) < x ? nextafterf(f, INFINITY) : f;
    };
    P.inv_beta2_up_f = f_up(P.inv_beta2_up);
    P.inv_k_up_f = f_up(P.inv_k_up);
    P.f32_bounds = std::isfinite(P.inv_beta2_up_f) && HP_PLAN_F32;
    return P;
}

// Plan (warp per ray) -> scan of the exact-region sizes -> (host reads the
// total) -> expand (slot -> ray) -> exact evaluation (thread per candidate).
template <class BestT>
int launch_exact(const Csr& C, const Params& P, SampleWs& w, cudaStream_t s) {
    {
        if (cudaMemsetAsync(w.work, 0, 3 * sizeof(unsigned long long), s) != cudaSuccess)
            return cuda_status(cudaGetLastError(), "k_sample_plan memset");
        TimedSpan ts("k_sample_plan", s);
        k_sample_plan<<<device_sms() * 8, kThreads, 0, s>>>(C, P, w.plan, w.eoff, w.work);
        HP_CHECK_LAUNCH("k_sample_plan");
    }
    HP_TRY(exclusive_scan_i64(w.eoff, w.eoff, C.m, w.scan, s));
    // no host round trip: the kernels read the exact-region total on the
    // device and do nothing if it exceeds the capacity (reported in r_off[m])
    {
        TimedSpan ts("k_sample_expand", s);
        k_sample_expand<<<grid_for(C.m, 256), 256, 0, s>>>(C.m, w.eoff, w.x.ray, w.x.cap);
        HP_CHECK_LAUNCH("k_sample_expand");
    }
    {
        TimedSpan ts("k_sample_exact", s);
        if (P.emit_knn)
            k_sample_exact<BestT, true><<<device_sms() * 16, kThreads, 0, s>>>(C, P, w.plan, w.eoff, w.x, w.work + 2);
        else
            k_sample_exact<BestT, false><<<device_sms() * 16, kThreads, 0, s>>>(C, P, w.plan, w.eoff, w.x, w.work + 2);
        HP_CHECK_LAUNCH("k_sample_exact");
    }
    return HP_OK;
}

int dispatch_exact(const Csr& C, const Params& P, SampleWs& w, cudaStream_t s) {
    if (P.K <= 8) return launch_exact<Best<8>>(C, P, w, s);
    if (P.K <= 32) return launch_exact<Best<32>>(C, P, w, s);
    return launch_exact<BestDyn>(C, P, w, s);
}

int launch_retain(const Csr& C, const Params& P, const RayOut& RO, const SampleWs& w, cudaStream_t s) {
    TimedSpan ts("k_sample_retain", s);
#if HP_RETAIN_SHORT > 0
    // short rays one thread each; the rest one warp each (the list's length
    // stays on the device: a fixed grid strides over it)
    const int gshort = grid_for(C.m, kThreads);
    const int glong = device_sms() * 8;
    if (P.emit_knn) {
        k_sample_retain_short<true><<<gshort, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x, w.longs, w.work + 1);
        k_sample_retain_long<true><<<glong, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x, w.longs, w.work + 1);
    } else {
        k_sample_retain_short<false><<<gshort, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x, w.longs, w.work + 1);
        k_sample_retain_long<false><<<glong, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x, w.longs, w.work + 1);
    }
#else
    // one ray per warp: as many warps in flight as the SMs hold (latency-bound)
    const int64_t blocks = (C.m + kWarps - 1) / kWarps;
    const int grid = int(blocks < (1 << 30) ? blocks : (1 << 30));
    if (P.emit_knn)
        k_sample_retain<true><<<grid, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x);
    else
        k_sample_retain<false><<<grid, kThreads, 0, s>>>(C, P, RO, w.plan, w.eoff, w.x);
#endif
    HP_CHECK_LAUNCH("k_sample_retain");
    return HP_OK;
}

int launch_emit(const Csr& C, const Params& P, const int64_t* r_off, const SampleWs& w, const Outputs& O,
                cudaStream_t s) {
    TimedSpan ts("k_emit", s);
    const int64_t m = C.m;
#if HP_EMIT_FLAT
    if (P.emit_knn)
        k_emit_flat<true><<<grid_for(m, 256), 256, 0, s>>>(C, P, r_off, w.eoff, w.x, O);
    else
        k_emit_flat<false><<<grid_for(m, 256), 256, 0, s>>>(C, P, r_off, w.eoff, w.x, O);
    HP_CHECK_LAUNCH("k_emit");
    return HP_OK;
#endif
    // one warp per ray (a thread per short ray measured slower: its writes do not coalesce)
    if (P.emit_knn)
        k_emit<true><<<grid_for(m * 32, 256), 256, 0, s>>>(C, P, r_off, w.eoff, w.x, O);
    else
        k_emit<false><<<grid_for(m * 32, 256), 256, 0, s>>>(C, P, r_off, w.eoff, w.x, O);
    HP_CHECK_LAUNCH("k_emit");
    return HP_OK;
}

int validate(const hp_sampler_params* p, const double* colors, int64_t n_colors) {
    if (!p || p->k_neighbors < 1 || p->k_neighbors > HP_MAX_K) {
        set_error("k_neighbors must be in [1, %d] on the device path", HP_MAX_K);
        return HP_EINVAL;
    }
    if (p->want_color && !colors && n_colors > 0) {
        set_error("want_color set but colors is NULL");
        return HP_EINVAL;
    }
    return HP_OK;
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_sample_workspace_bytes(int64_t m, int64_t total, int64_t exact_capacity,
                                         const hp_sampler_params* p, size_t* bytes) {
    Carver c(nullptr, 0);
    carve_sample(c, m, exact_capacity, p && p->want_color, p && p->emit_knn ? p->k_neighbors : 0);
    *bytes = c.used + 256;
    (void)total;
    return HP_OK;
}

extern "C" int hp_sample_run(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                             const double* dist, int64_t total, int64_t exact_capacity, const double* slopes,
                             const int32_t* query_facts, const hp_sampler_params* p, const double* colors,
                             int64_t n_colors, int64_t* r_off, double* t_end, void* workspace,
                             size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    (void)total;
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, exact_capacity, p->want_color, p->emit_knn ? p->k_neighbors : 0);
    if (!c.ok()) {
        set_error("hp_sample_run: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Csr C{offsets, ids, t, dist, slopes, colors, m, query_facts};
    Params P = to_params(p);
    if (m > 0) {
        HP_TRY(dispatch_exact(C, P, w, s));
        HP_TRY(launch_retain(C, P, RayOut{r_off, t_end}, w, s));
    }
    HP_TRY(exclusive_scan_i64(r_off, r_off, m, w.scan, s));
    if (m > 0) {
        k_mark_exact_overflow<<<1, 1, 0, s>>>(w.eoff + m, exact_capacity, r_off + m);
        HP_CHECK_LAUNCH("k_mark_exact_overflow");
    }
    return HP_OK;
}

// Prefix mode (hp_query_prefix): the same passes over each ray's sorted
// prefix; rays whose work may reach past it are flagged instead.
extern "C" int hp_sample_run_prefix(const int64_t* offsets, int64_t m, const hp_sample_prefix* pre,
                                    int64_t exact_capacity, const double* slopes, const int32_t* query_facts,
                                    const hp_sampler_params* p, const double* colors, int64_t n_colors,
                                    int64_t* r_off, double* t_end, int32_t* flagged, void* workspace,
                                    size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    if (!pre || !flagged || (m > 0 && (!pre->start || !pre->length || !pre->cut_t || !pre->cut_d || !query_facts))) {
        set_error("hp_sample_run_prefix: the prefix arrays, facts and flagged are required");
        return HP_EINVAL;
    }
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, exact_capacity, p->want_color, p->emit_knn ? p->k_neighbors : 0);
    if (!c.ok()) {
        set_error("hp_sample_run_prefix: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(flagged + m, 0, sizeof(int32_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_sample_run_prefix memset");
    Csr C{offsets, nullptr, pre->t, pre->dist, slopes, colors, m, query_facts,
          pre->start, pre->length, pre->ids, pre->cut_t, pre->cut_d, flagged, pre->u};
    Params P = to_params(p);
    if (m > 0) {
        HP_TRY(dispatch_exact(C, P, w, s));
        HP_TRY(launch_retain(C, P, RayOut{r_off, t_end}, w, s));
    }
    HP_TRY(exclusive_scan_i64(r_off, r_off, m, w.scan, s));
    if (m > 0) {
        k_mark_exact_overflow<<<1, 1, 0, s>>>(w.eoff + m, exact_capacity, r_off + m);
        HP_CHECK_LAUNCH("k_mark_exact_overflow");
    }
    return HP_OK;
}

extern "C" int hp_sample_emit_prefix(const int64_t* offsets, int64_t m, const hp_sample_prefix* pre,
                                     int64_t exact_capacity, const double* slopes, const hp_sampler_params* p,
                                     const double* colors, int64_t n_colors, const int64_t* r_off, int64_t R,
                                     int64_t* r_id, double* r_t, double* r_dist, double* r_udf, double* r_alpha,
                                     double* r_w, double* r_color, int64_t* r_knn_id, double* r_knn_w,
                                     void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    if (!pre) {
        set_error("hp_sample_emit_prefix: prefix is NULL");
        return HP_EINVAL;
    }
    if (R == 0 || m == 0) return HP_OK;
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, exact_capacity, p->want_color, p->emit_knn ? p->k_neighbors : 0);
    if (!c.ok()) {
        set_error("hp_sample_emit_prefix: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Csr C{offsets, nullptr, pre->t, pre->dist, slopes, colors, m, nullptr,
          pre->start, pre->length, pre->ids, pre->cut_t, pre->cut_d, nullptr};
    Params P = to_params(p);
    Outputs O{r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, r_knn_id, r_knn_w};
    if (P.emit_knn && (!r_knn_id || !r_knn_w)) {
        set_error("emit_knn set but r_knn_id / r_knn_w is NULL");
        return HP_EINVAL;
    }
    return launch_emit(C, P, r_off, w, O, s);
}

extern "C" int hp_sample_emit(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                              const double* dist, int64_t total, int64_t exact_capacity,
                              const double* slopes, const hp_sampler_params* p, const double* colors,
                              int64_t n_colors, const int64_t* r_off, int64_t R, int64_t* r_id, double* r_t,
                              double* r_dist, double* r_udf, double* r_alpha, double* r_w, double* r_color,
                              int64_t* r_knn_id, double* r_knn_w, void* workspace, size_t workspace_bytes,
                              hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    (void)total;
    if (R == 0 || m == 0) return HP_OK;
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, exact_capacity, p->want_color, p->emit_knn ? p->k_neighbors : 0);
    if (!c.ok()) {
        set_error("hp_sample_emit: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Csr C{offsets, ids, t, dist, slopes, colors, m, nullptr};
    Params P = to_params(p);
    Outputs O{r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color, r_knn_id, r_knn_w};
    if (P.emit_knn && (!r_knn_id || !r_knn_w)) {
        set_error("emit_knn set but r_knn_id / r_knn_w is NULL");
        return HP_EINVAL;
    }
    return launch_emit(C, P, r_off, w, O, s);
}

namespace hp {
namespace {
// a warp per 32 consecutive output rays, rows copied with the flat lane map
// of k_emit_flat (coalesced writes)
__global__ void k_splice(int64_t m, const int64_t* __restrict__ off_out, const int64_t* __restrict__ r_off,
                         const int64_t* __restrict__ s_off, const int64_t* __restrict__ pos, int K,
                         hp_sample_fields A, hp_sample_fields B, hp_sample_fields O) {
    const int lane = lane_id();
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r0 = (blockIdx.x * int64_t(blockDim.x >> 5) + warp_id()) * 32; r0 < m; r0 += warps * 32) {
        const int64_t r = r0 + lane;
        int n = 0, sub = 0;
        int64_t src = 0;
        if (r < m) {
            n = int(off_out[r + 1] - off_out[r]);
            const int64_t p = pos[r];
            sub = p >= 0;
            src = sub ? s_off[p] : r_off[r];
        }
        const int64_t o0 = __shfl_sync(0xffffffffu, r < m ? off_out[r] : 0, 0);
        const int incl = warp_incl_scan(n);
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int b0 = 0; b0 < total; b0 += 32) {
            const int sidx = b0 + lane;
            int owner = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, owner + step - 1);
                if (v <= sidx) owner += step;
            }
            const int excl = __shfl_sync(0xffffffffu, incl - n, owner);
            const int64_t so = __shfl_sync(0xffffffffu, src, owner);
            const int fs = __shfl_sync(0xffffffffu, sub, owner);
            if (sidx >= total) continue;
            const hp_sample_fields& S = fs ? B : A;
            const int64_t i = so + (sidx - excl), o = o0 + sidx;
            O.r_id[o] = S.r_id[i];
            O.r_t[o] = S.r_t[i];
            O.r_dist[o] = S.r_dist[i];
            O.r_udf[o] = S.r_udf[i];
            O.r_alpha[o] = S.r_alpha[i];
            O.r_w[o] = S.r_w[i];
            if (O.r_color)
                for (int x = 0; x < 3; x++) O.r_color[3 * o + x] = S.r_color[3 * i + x];
            if (O.r_knn_id)
                for (int b = 0; b < K; b++) {
                    O.r_knn_id[o * K + b] = S.r_knn_id[i * K + b];
                    O.r_knn_w[o * K + b] = S.r_knn_w[i * K + b];
                }
        }
    }
}
}  // namespace
}  // namespace hp

extern "C" int hp_splice_samples(int64_t m, const int64_t* off_out, const int64_t* r_off, const int64_t* s_off,
                                 const int64_t* pos, int32_t k_neighbors, const hp_sample_fields* main_rows,
                                 const hp_sample_fields* sub_rows, const hp_sample_fields* out, hp_stream_t stream) {
    if (m < 0 || !main_rows || !sub_rows || !out || (m > 0 && (!off_out || !r_off || !s_off || !pos)) ||
        k_neighbors < 0 || (out->r_knn_id && k_neighbors < 1)) {
        set_error("hp_splice_samples: invalid arguments");
        return HP_EINVAL;
    }
    if (m == 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    TimedSpan ts("k_splice", s);
    k_splice<<<grid_for(m, 256), 256, 0, s>>>(m, off_out, r_off, s_off, pos, k_neighbors, *main_rows, *sub_rows,
                                               *out);
    HP_CHECK_LAUNCH("k_splice");
    return HP_OK;
}

extern "C" int hp_primary_surface(const int64_t* r_off, int64_t m, const int64_t* r_id, const double* r_t,
                                  int64_t* primary_id, double* primary_t, hp_stream_t stream) {
    if (m <= 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_primary<<<grid_for(m, 256), 256, 0, s>>>(r_off, m, r_id, r_t, primary_id, primary_t);
    HP_CHECK_LAUNCH("k_primary");
    return HP_OK;
}

extern "C" int hp_csr_stats(const int64_t* offsets, int64_t m, int64_t* out2, hp_stream_t stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(out2, 0, 2 * sizeof(int64_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_csr_stats memset");
    k_csr_stats<<<grid_for(m > 0 ? m : 1, 256, 148 * 4), 256, 0, s>>>(offsets, m, out2);
    HP_CHECK_LAUNCH("k_csr_stats");
    return HP_OK;
}

extern "C" int hp_sample_debug_counters(int64_t* out8, int reset) {
    unsigned long long h[8];
    cudaError_t e = cudaMemcpyFromSymbol(h, g_dbg, sizeof(h));
    if (e != cudaSuccess) return cuda_status(e, "hp_sample_debug_counters");
    for (int k = 0; k < 8; k++) out8[k] = int64_t(h[k]);
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        e = cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
        if (e != cudaSuccess) return cuda_status(e, "hp_sample_debug_counters");
    }
    return HP_OK;
}
