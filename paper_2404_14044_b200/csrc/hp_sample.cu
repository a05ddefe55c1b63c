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
// Exact reformulations (bit-identical selections):
//   * use_el(j) = (#{ds_i <= r_j} >= K) is monotone in j when t is sorted and
//     slope >= 0, so one binary search over j replaces the per-j count.
//   * K-nearest search: candidates are cut into blocks of 32 consecutive (in
//     t) elements, each block sorted by (ds, i).  The search visits blocks
//     outward from j in order of the lower bound (t_edge - t_j)^2 and scans a
//     block only while ds^2 (a lower bound of d2) can still beat the K-th best.
//     Selection key (d2, i) reproduces the reference's strict-< insertion.
//   * early exit: once retention is decided (T < eps, or T < tau_min) and, in
//     exact-t_end mode, T has underflowed to exactly 0.0 (then every later
//     product stays 0), the remaining candidates cannot change any output.
// Rays violating the preconditions (unsorted t, negative/NaN values) fall
// back to the reference's direct O(q^2) loops on the device.
#include <math_constants.h>

#include <cfloat>
#include <climits>

#include "hp_common.cuh"

namespace hp {
namespace {

constexpr int kThreads = 128;
constexpr int kSmemCap = 2048;  // candidates staged in shared memory per ray
constexpr int kRetCap = 64;     // retained candidates buffered per ray

// Path counters (rays, fast rays, proved-zero rays, exact evals, candidates,
// bound evals); read with hp_sample_debug_counters().
__device__ unsigned long long g_dbg[8];

struct Params {
    int K;
    int eps_mode, want_color, exact_t_end;
    double beta2, gamma, eps, tau_min;
};

struct Csr {
    const int64_t* off;
    const int64_t* ids;
    const double* t;
    const double* ds;
    const double* slopes;
    const double* colors;
    int64_t m;
    int64_t max_q;  // longest segment (sizes the per-CTA scratch of long rays)
};

struct Stage {  // retained candidates between hp_sample_run and hp_sample_emit
    int32_t* j;
    double* udf;
    double* alpha;
    double* w;
    double* col;  // [cap, 3]
    int64_t cap;
};

struct Outputs {
    int64_t* r_id;
    double *r_t, *r_dist, *r_udf, *r_alpha, *r_w, *r_color;
};

__device__ __forceinline__ bool kless(double d2a, int ia, double d2b, int ib) {
    return d2a < d2b || (d2a == d2b && ia < ib);
}

// K-best list in registers (MAXK compile-time, ksel <= MAXK at runtime),
// ascending by (d2, i).
template <int MAXK>
struct Best {
    double d[MAXK];
    int i[MAXK];
    __device__ __forceinline__ void init(int ksel) {
#pragma unroll
        for (int b = 0; b < MAXK; b++) {
            d[b] = CUDART_INF;
            i[b] = INT_MAX;
        }
        (void)ksel;
    }
    __device__ __forceinline__ double kth_d(int ksel) const {
        double v = d[0];
#pragma unroll
        for (int b = 0; b < MAXK; b++)
            if (b == ksel - 1) v = d[b];
        return v;
    }
    __device__ __forceinline__ int kth_i(int ksel) const {
        int v = i[0];
#pragma unroll
        for (int b = 0; b < MAXK; b++)
            if (b == ksel - 1) v = i[b];
        return v;
    }
    template <class F>
    __device__ __forceinline__ void for_each(int ksel, F f) const {
#pragma unroll
        for (int b = 0; b < MAXK; b++)
            if (b < ksel) f(d[b], i[b]);
    }
    // caller guarantees (nd, ni) < the current ksel-th entry
    __device__ __forceinline__ void insert(int ksel, double nd, int ni) {
        bool placed = false;
#pragma unroll
        for (int b = MAXK - 1; b >= 1; --b) {
            if (b < ksel && !placed) {
                if (kless(nd, ni, d[b - 1], i[b - 1])) {
                    d[b] = d[b - 1];
                    i[b] = i[b - 1];
                } else {
                    d[b] = nd;
                    i[b] = ni;
                    placed = true;
                }
            }
        }
        if (!placed) {
            d[0] = nd;
            i[0] = ni;
        }
    }
};

// Large-K variant: arrays in local memory, dynamic loops.
struct BestDyn {
    double d[HP_MAX_K];
    int i[HP_MAX_K];
    __device__ void init(int ksel) {
        for (int b = 0; b < ksel; b++) {
            d[b] = CUDART_INF;
            i[b] = INT_MAX;
        }
    }
    template <class F>
    __device__ void for_each(int ksel, F f) const {
        for (int b = 0; b < ksel; b++) f(d[b], i[b]);
    }
    __device__ double kth_d(int ksel) const { return d[ksel - 1]; }
    __device__ int kth_i(int ksel) const { return i[ksel - 1]; }
    __device__ void insert(int ksel, double nd, int ni) {
        int b = ksel - 1;
        while (b > 0 && kless(nd, ni, d[b - 1], i[b - 1])) {
            d[b] = d[b - 1];
            i[b] = i[b - 1];
            b--;
        }
        d[b] = nd;
        i[b] = ni;
    }
};

struct RaySmem {
    double t[kSmemCap];
    double ds[kSmemCap];
    double bds[kSmemCap];
    int bidx[kSmemCap];
    double ca[kThreads], cd[kThreads], ccol[kThreads * 3];
    // retained buffer
    int rj[kRetCap];
    double rudf[kRetCap], ralpha[kRetCap], rw[kRetCap], rcol[kRetCap * 3];
    int red[kThreads / 32 + 1];
    int flag;
    int nret;
    int stop;
    int jstar;
    int je, jz;
    double T, U, dsk, exit_T;
    int64_t stage_at;
};

// Per-candidate evaluation: udf, alpha (and colour) of candidate j.
template <class BestT>
__device__ void eval_candidate(const double* __restrict__ T, const double* __restrict__ DS,
                               const double* __restrict__ BDS, const int* __restrict__ BIDX, int q,
                               int j, bool fast, int jstar, double slope, const Params& P,
                               const int64_t* __restrict__ ids_ray, const double* __restrict__ colors,
                               double& udf, double& alpha, double* col3) {
    const double tj = T[j];
    const double rj = dmul(slope, tj);
    BestT best;
    bool use_el;
    int ksel;
    if (fast) {
        use_el = j >= jstar;
        ksel = use_el ? P.K : (q < P.K ? q : P.K);
    } else {
        int n_el = 0;
        for (int i = 0; i < q; i++) n_el += (DS[i] <= rj);
        use_el = n_el >= P.K;
        const int pool = use_el ? n_el : q;
        ksel = pool > P.K ? P.K : pool;
    }
    best.init(ksel);
    double kd = CUDART_INF;
    int ki = INT_MAX;
    if (fast) {
        const int nblk = (q + 31) >> 5;
        const int B = j >> 5;
        auto scan_block = [&](int b) {
            const int e0 = b << 5, e1 = (e0 + 32 < q) ? e0 + 32 : q;
            for (int e = e0; e < e1; e++) {
                const double di = BDS[e];
                if (use_el && di > rj) break;
                const double di2 = dmul(di, di);
                if (di2 > kd) break;
                const int i = BIDX[e];
                const double dt = dsub(T[i], tj);
                const double d2 = dadd(dmul(dt, dt), di2);
                if (kless(d2, i, kd, ki)) {
                    best.insert(ksel, d2, i);
                    kd = best.kth_d(ksel);
                    ki = best.kth_i(ksel);
                }
            }
        };
        scan_block(B);
        int left = B - 1, right = B + 1;
        for (;;) {
            double lbl = CUDART_INF, lbr = CUDART_INF;
            if (left >= 0) {
                const double dt = dsub(T[(left << 5) + 31], tj);
                lbl = dmul(dt, dt);
            }
            if (right < nblk) {
                const double dt = dsub(T[right << 5], tj);
                lbr = dmul(dt, dt);
            }
            const bool goleft = lbl <= lbr;
            const double lb = goleft ? lbl : lbr;
            if (!(lb <= kd) || (left < 0 && right >= nblk)) break;
            if (goleft) {
                scan_block(left);
                left--;
            } else {
                scan_block(right);
                right++;
            }
        }
    } else {
        for (int i = 0; i < q; i++) {  // reference loop (_kernels.py:607-620)
            const double di = DS[i];
            if (use_el && di > rj) continue;
            const double dt = dsub(T[i], tj);
            const double d2 = dadd(dmul(dt, dt), dmul(di, di));
            if (d2 < kd) {
                best.insert(ksel, d2, i);
                kd = best.kth_d(ksel);
                ki = best.kth_i(ksel);
            }
        }
    }
    double acc = 0.0;
    best.for_each(ksel, [&](double d2, int) { acc = dadd(acc, sqrt(d2)); });
    udf = __ddiv_rn(acc, double(ksel));
    alpha = dmul(P.gamma, exp(__ddiv_rn(-dmul(udf, udf), P.beta2)));
    if (P.want_color) {
        int nz = 0;
        best.for_each(ksel, [&](double d2, int) { nz += (d2 == 0.0); });
        double c0 = 0.0, c1 = 0.0, c2 = 0.0;
        if (nz > 0) {
            best.for_each(ksel, [&](double d2, int i) {
                if (d2 != 0.0) return;
                const int64_t pid = ids_ray[i];
                c0 = dadd(c0, colors[3 * pid]);
                c1 = dadd(c1, colors[3 * pid + 1]);
                c2 = dadd(c2, colors[3 * pid + 2]);
            });
            c0 = __ddiv_rn(c0, double(nz));
            c1 = __ddiv_rn(c1, double(nz));
            c2 = __ddiv_rn(c2, double(nz));
        } else {
            double wsum = 0.0;
            best.for_each(ksel, [&](double d2, int i) {
                const double wgt = __ddiv_rn(1.0, sqrt(d2));
                const int64_t pid = ids_ray[i];
                c0 = dadd(c0, dmul(wgt, colors[3 * pid]));
                c1 = dadd(c1, dmul(wgt, colors[3 * pid + 1]));
                c2 = dadd(c2, dmul(wgt, colors[3 * pid + 2]));
                wsum = dadd(wsum, wgt);
            });
            c0 = __ddiv_rn(c0, wsum);
            c1 = __ddiv_rn(c1, wsum);
            c2 = __ddiv_rn(c2, wsum);
        }
        col3[0] = c0;
        col3[1] = c1;
        col3[2] = c2;
    }
}

// Sort the 32-element block (in t order) of every lane-group by (ds, i):
// one warp per block, bitonic network over shuffles.
__device__ void build_blocks(const double* __restrict__ DS, double* __restrict__ BDS, int* __restrict__ BIDX,
                             int q) {
    const int nblk = (q + 31) >> 5;
    const int lane = lane_id();
    for (int b = warp_id(); b < nblk; b += kThreads / 32) {
        const int e = (b << 5) + lane;
        double k = e < q ? DS[e] : CUDART_INF;
        int id = e < q ? e : INT_MAX;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                const double ok = __shfl_xor_sync(0xffffffffu, k, stride);
                const int oid = __shfl_xor_sync(0xffffffffu, id, stride);
                const bool ascending = (lane & size) == 0;
                const bool lower = (lane & stride) == 0;
                // ascending block: the lower lane keeps the smaller key
                const bool take = (lower == ascending) ? kless(ok, oid, k, id) : kless(k, id, ok, oid);
                if (take) {
                    k = ok;
                    id = oid;
                }
            }
        }
        if (e < q) {
            BDS[e] = k;
            BIDX[e] = id;
        }
    }
}

// Upper bound of the reference's factor fl(1 - alpha_j) for candidate j
// (DESIGN.md "sampler: transmittance bound").  Any ksel members of j's pool
// give a mean distance >= the K-nearest mean, so the udf bound is the mean
// over the ksel pool members nearest to j in t order, inflated by 1e-12 (which
// dominates every fp64 rounding of the two sums); alpha is then bounded
// below with a further 1e-12 margin (covers exp() ulp differences).  All
// operations used afterwards are monotone, so the chain U_{j+1} = U_j * u_j
// evaluated in the reference's order dominates its transmittance T_j.
__device__ double bound_factor(const double* __restrict__ T, const double* __restrict__ DS, int q, int j,
                               int jstar, double slope, const Params& P) {
    const double tj = T[j];
    const double rj = dmul(slope, tj);
    const bool use_el = j >= jstar;
    const int ksel = use_el ? P.K : (q < P.K ? q : P.K);
    double sum = 0.0;
    int found = 0;
    int l = j, r = j + 1;
    while (found < ksel) {
        int i;
        if (l < 0) {
            i = r++;
        } else if (r >= q) {
            i = l--;
        } else if (dsub(tj, T[l]) <= dsub(T[r], tj)) {
            i = l--;
        } else {
            i = r++;
        }
        const double di = DS[i];
        if (use_el && di > rj) continue;
        const double dt = dsub(T[i], tj);
        sum = dadd(sum, sqrt(dadd(dmul(dt, dt), dmul(di, di))));
        found++;
    }
    const double udf_up = __ddiv_rn(dmul(sum, 1.0 + 1e-12), double(ksel));
    const double a_lo = dmul(dmul(P.gamma, exp(__ddiv_rn(-dmul(udf_up, udf_up), P.beta2))), 1.0 - 1e-12);
    return dsub(1.0, a_lo);
}

// K-th smallest ds over the ray (ds >= 0), from the (ds, i)-sorted 32-blocks:
// warp 0 pops the smallest block head K times.  Returns +inf if q < K.
__device__ double kth_smallest_ds(const double* __restrict__ BDS, int q, int K) {
    if (q < K) return CUDART_INF;
    const int nblk = (q + 31) >> 5;
    // each lane owns blocks lane, lane+32, ... ; head pointer per block kept in
    // registers for up to 4 blocks per lane (q <= 4096), else generic loop
    int head[4] = {0, 0, 0, 0};
    double v = 0.0;
    const int lane = lane_id();
    for (int k = 0; k < K; k++) {
        double best = CUDART_INF;
        int bb = -1;
#pragma unroll
        for (int s = 0; s < 4; s++) {
            const int b = lane + 32 * s;
            if (b < nblk) {
                const int e = (b << 5) + head[s];
                const int e_end = min((b << 5) + 32, q);
                if (e < e_end && BDS[e] < best) {
                    best = BDS[e];
                    bb = s;
                }
            }
        }
        // warp argmin (value, lane)
        double mv = best;
        int ml = lane;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, mv, o);
            const int ol = __shfl_xor_sync(0xffffffffu, ml, o);
            if (ov < mv || (ov == mv && ol < ml)) {
                mv = ov;
                ml = ol;
            }
        }
        if (lane == ml && bb >= 0) head[bb]++;
        v = mv;
    }
    return v;
}

// One ray, block-wide.  mode 0: stage retained candidates; mode 1: write them
// directly to the outputs at r_off[ray].
//
// Fast path (t sorted, ds >= 0, slope >= 0):
//   1. bound chain U over candidates (cheap factors) -> Je = first j with
//      U_j < thr (retention is decided before Je) and whether U reaches 0
//      (then the exact transmittance is exactly 0).
//   2. exact udf/alpha (block K-nearest search) for j < Je -- or for all j
//      when the exact t_end is requested and U never reached 0 -- with the
//      reference's sequential compositing and retention.
// Slow path: exact evaluation of every candidate with the reference loops.
template <class BestT>
__device__ void sample_ray(RaySmem& S, const Csr& C, const Params& P, int64_t ray, int mode,
                           double* __restrict__ gscratch_ds, int* __restrict__ gscratch_idx,
                           int64_t* __restrict__ rcount, double* __restrict__ t_end,
                           int64_t* __restrict__ ray_stage, int64_t* __restrict__ stage_cursor,
                           const Stage& ST, int* __restrict__ ovf_list, int* __restrict__ ovf_n,
                           const int64_t* __restrict__ r_off, const Outputs& O) {
    const int tid = threadIdx.x;
    const int64_t lo = C.off[ray];
    const int q = int(C.off[ray + 1] - lo);
    if (q == 0) {
        if (mode == 0 && tid == 0) {
            rcount[ray] = 0;
            t_end[ray] = 1.0;
            ray_stage[ray] = 0;
        }
        return;
    }
    const double slope = C.slopes[ray];
    const bool in_smem = q <= kSmemCap;
    const double* T;
    const double* DS;
    double* BDS;
    int* BIDX;
    if (in_smem) {
        for (int k = tid; k < q; k += kThreads) {
            S.t[k] = C.t[lo + k];
            S.ds[k] = C.ds[lo + k];
        }
        T = S.t;
        DS = S.ds;
        BDS = S.bds;
        BIDX = S.bidx;
    } else {
        T = C.t + lo;
        DS = C.ds + lo;
        BDS = gscratch_ds + int64_t(blockIdx.x) * C.max_q;
        BIDX = gscratch_idx + int64_t(blockIdx.x) * C.max_q;
    }
    __syncthreads();  // staged t/ds visible to the whole block
    // fast-path preconditions: t finite and non-decreasing, ds finite and >= 0
    bool ok = true;
    for (int k = tid; k < q; k += kThreads) {
        const double tk = T[k], dk = DS[k];
        ok &= (fabs(tk) <= DBL_MAX) && (dk >= 0.0) && (dk <= DBL_MAX);
        if (k + 1 < q) ok &= !(T[k + 1] < tk);
    }
    const bool fast = __syncthreads_and(ok) && slope >= 0.0 && slope <= DBL_MAX;
    const double thr = P.eps_mode ? P.eps : P.tau_min;
    if (fast) {
        build_blocks(DS, BDS, BIDX, q);
        __syncthreads();
        if (P.K <= 32 && q <= 4096) {
            if (warp_id() == 0) {
                const double dsk = kth_smallest_ds(BDS, q, P.K);
                if (lane_id() == 0) S.dsk = dsk;
            }
            __syncthreads();
            // jstar = first j with slope * t_j >= ds_(K)   (r_j is monotone)
            if (tid == 0) {
                int a = 0, b = q;
                const double dsk = S.dsk;
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (dmul(slope, T[mid]) >= dsk) b = mid; else a = mid + 1;
                }
                S.jstar = (dsk <= DBL_MAX) ? a : q;
            }
        } else {
            // generic: binary search on j with block-wide counts
            int a = 0, b = q;
            while (a < b) {
                const int mid = (a + b) >> 1;
                const double rj = dmul(slope, T[mid]);
                int c = 0;
                for (int k = tid; k < q; k += kThreads) c += (DS[k] <= rj);
                c = warp_sum(c);
                if (lane_id() == 0) S.red[warp_id()] = c;
                __syncthreads();
                int tot = 0;
#pragma unroll
                for (int w = 0; w < kThreads / 32; w++) tot += S.red[w];
                __syncthreads();
                if (tot >= P.K) b = mid; else a = mid + 1;
            }
            if (tid == 0) S.jstar = a;
        }
        if (tid == 0) {
            S.U = 1.0;
            S.je = q;
            S.jz = 0;  // 1 when the bound chain reached exactly 0
        }
        __syncthreads();
        // ---- 1. bound chain
        const int jstar = S.jstar;
        for (int c0 = 0; c0 < q; c0 += kThreads) {
            const int j = c0 + tid;
            if (j < q) S.ca[tid] = bound_factor(T, DS, q, j, jstar, slope, P);
            __syncthreads();
            if (tid == 0) {
                double U = S.U;
                int je = S.je, jz = 0;
                const int c1 = min(c0 + kThreads, q);
                for (int jj = c0; jj < c1; jj++) {
                    if (je == q && U < thr) je = jj;
                    U = dmul(U, S.ca[jj - c0]);
                    if (U == 0.0) {
                        jz = 1;
                        if (je == q && thr > 0.0) je = jj + 1;  // U_{jj+1} = 0 < thr
                        break;
                    }
                }
                S.U = U;
                S.je = je;
                S.jz = jz;
                S.stop = jz || (!P.exact_t_end && je < q);
            }
            __syncthreads();
            if (S.stop) break;
        }
    } else if (tid == 0) {
        S.je = q;
        S.jz = 0;
    }
    __syncthreads();
    // exact region: [0, E)
    const int je = S.je;
    const bool proved_zero = fast && S.jz;
    const int E = (P.exact_t_end && !proved_zero) ? q : je;
    const int jstar = fast ? S.jstar : 0;
    if (tid == 0 && mode == 0) {
        atomicAdd(&g_dbg[0], 1ull);
        atomicAdd(&g_dbg[1], fast ? 1ull : 0ull);
        atomicAdd(&g_dbg[2], proved_zero ? 1ull : 0ull);
        atomicAdd(&g_dbg[3], (unsigned long long)E);
        atomicAdd(&g_dbg[4], (unsigned long long)q);
        atomicAdd(&g_dbg[5], (unsigned long long)(fast ? S.jstar : -1));
    }
    if (tid == 0) {
        S.nret = 0;
        S.T = 1.0;
        S.stop = 0;
        S.exit_T = -1.0;
    }
    __syncthreads();
    const int64_t* ids_ray = C.ids + lo;
    int64_t out_base = 0;
    if (mode == 1) out_base = r_off[ray];
    for (int c0 = 0; c0 < E; c0 += kThreads) {
        const int j = c0 + tid;
        if (j < E) {
            double u, a;
            eval_candidate<BestT>(T, DS, BDS, BIDX, q, j, fast, jstar, slope, P, ids_ray, C.colors, u, a,
                                  &S.ccol[3 * tid]);
            S.cd[tid] = u;
            S.ca[tid] = a;
        }
        __syncthreads();
        if (tid == 0) {
            // sequential front-to-back compositing (_kernels.py:661-697)
            double Tr = S.T;
            int nret = S.nret;
            const int c1 = min(c0 + kThreads, E);
            int stop = 0;
            for (int jj = c0; jj < c1; jj++) {
                const int k = jj - c0;
                if (!P.exact_t_end && Tr < thr) {  // exit mode: retention decided
                    S.exit_T = Tr;
                    stop = 1;
                    break;
                }
                const double a = S.ca[k];
                const double w = dmul(a, Tr);
                const bool keep = P.eps_mode ? (w >= P.eps) : !(Tr < P.tau_min);
                if (keep) {
                    if (mode == 1) {
                        const int64_t o = out_base + nret;
                        O.r_id[o] = ids_ray[jj];
                        O.r_t[o] = T[jj];
                        O.r_dist[o] = DS[jj];
                        O.r_udf[o] = S.cd[k];
                        O.r_alpha[o] = a;
                        O.r_w[o] = w;
                        if (P.want_color) {
                            O.r_color[3 * o] = S.ccol[3 * k];
                            O.r_color[3 * o + 1] = S.ccol[3 * k + 1];
                            O.r_color[3 * o + 2] = S.ccol[3 * k + 2];
                        }
                    } else if (nret < kRetCap) {
                        S.rj[nret] = jj;
                        S.rudf[nret] = S.cd[k];
                        S.ralpha[nret] = a;
                        S.rw[nret] = w;
                        if (P.want_color) {
                            S.rcol[3 * nret] = S.ccol[3 * k];
                            S.rcol[3 * nret + 1] = S.ccol[3 * k + 1];
                            S.rcol[3 * nret + 2] = S.ccol[3 * k + 2];
                        }
                    }
                    nret++;
                }
                Tr = dmul(Tr, dsub(1.0, a));
            }
            S.T = Tr;
            S.nret = nret;
            S.stop = stop;
        }
        __syncthreads();
        if (S.stop) break;
    }
    if (mode == 0) {
        if (tid == 0) {
            const int nret = S.nret;
            rcount[ray] = nret;
            double te;
            if (P.exact_t_end)
                te = proved_zero ? 0.0 : S.T;
            else
                te = S.exit_T >= 0.0 ? S.exit_T : S.T;
            t_end[ray] = te;
            int64_t st = -1;
            if (nret > 0 && nret <= kRetCap) {
                st = atomicAdd(reinterpret_cast<unsigned long long*>(stage_cursor), (unsigned long long)nret);
                if (st + nret > ST.cap) st = -1;
            } else if (nret == 0) {
                st = 0;
            }
            ray_stage[ray] = st;
            if (st < 0) ovf_list[atomicAdd(ovf_n, 1)] = int(ray);
            S.flag = int(st >= 0 && nret > 0);
            S.stage_at = st >= 0 ? st : 0;
        }
        __syncthreads();
        if (S.flag) {
            const int64_t st = S.stage_at;
            for (int k = tid; k < S.nret; k += kThreads) {
                ST.j[st + k] = S.rj[k];
                ST.udf[st + k] = S.rudf[k];
                ST.alpha[st + k] = S.ralpha[k];
                ST.w[st + k] = S.rw[k];
                if (P.want_color) {
                    ST.col[3 * (st + k)] = S.rcol[3 * k];
                    ST.col[3 * (st + k) + 1] = S.rcol[3 * k + 1];
                    ST.col[3 * (st + k) + 2] = S.rcol[3 * k + 2];
                }
            }
        }
    }
    __syncthreads();
}

template <class BestT>
__global__ void __launch_bounds__(kThreads) k_sample(Csr C, Params P, int mode, const int* __restrict__ ray_list,
                                                     const int* __restrict__ ray_list_n,
                                                     double* __restrict__ gscratch_ds, int* __restrict__ gscratch_idx,
                                                     int64_t* __restrict__ rcount, double* __restrict__ t_end,
                                                     int64_t* __restrict__ ray_stage, int64_t* __restrict__ stage_cursor,
                                                     Stage ST, int* __restrict__ ovf_list, int* __restrict__ ovf_n,
                                                     const int64_t* __restrict__ r_off, Outputs O) {
    extern __shared__ __align__(16) unsigned char dyn[];
    RaySmem& S = *reinterpret_cast<RaySmem*>(dyn);
    const int64_t n = ray_list ? int64_t(*ray_list_n) : C.m;
    for (int64_t k = blockIdx.x; k < n; k += gridDim.x) {
        const int64_t ray = ray_list ? int64_t(ray_list[k]) : k;
        sample_ray<BestT>(S, C, P, ray, mode, gscratch_ds, gscratch_idx, rcount, t_end, ray_stage, stage_cursor,
                          ST, ovf_list, ovf_n, r_off, O);
    }
}

// Copy staged retained candidates to the outputs (ray order).
__global__ void k_emit(Csr C, Params P, const int64_t* __restrict__ r_off, const int64_t* __restrict__ ray_stage,
                       Stage ST, Outputs O) {
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x >> 5) + warp_id(); r < C.m; r += warps) {
        const int64_t o = r_off[r], n = r_off[r + 1] - o, st = ray_stage[r];
        if (n == 0 || st < 0) continue;
        const int64_t lo = C.off[r];
        for (int64_t k = lane_id(); k < n; k += 32) {
            const int64_t j = lo + ST.j[st + k];
            O.r_id[o + k] = C.ids[j];
            O.r_t[o + k] = C.t[j];
            O.r_dist[o + k] = C.ds[j];
            O.r_udf[o + k] = ST.udf[st + k];
            O.r_alpha[o + k] = ST.alpha[st + k];
            O.r_w[o + k] = ST.w[st + k];
            if (P.want_color) {
                O.r_color[3 * (o + k)] = ST.col[3 * (st + k)];
                O.r_color[3 * (o + k) + 1] = ST.col[3 * (st + k) + 1];
                O.r_color[3 * (o + k) + 2] = ST.col[3 * (st + k) + 2];
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

struct SampleWs {
    int64_t* rcount;  // [m+1] -> scanned into r_off by the caller's array
    int64_t* ray_stage;
    int64_t* stage_cursor;
    int* ovf_list;
    int* ovf_n;
    Stage st;
    double* gds;
    int* gidx;
    void* scan;
};

constexpr int kSampleGrid = 148 * 2;

SampleWs carve_sample(Carver& c, int64_t m, int64_t total, int64_t cap, bool color, int64_t max_q) {
    const bool big = max_q > kSmemCap;
    (void)total;
    SampleWs w;
    w.rcount = nullptr;
    w.ray_stage = c.take<int64_t>(m > 0 ? m : 1);
    w.stage_cursor = c.take<int64_t>(1);
    w.ovf_list = c.take<int>(m > 0 ? m : 1);
    w.ovf_n = c.take<int>(1);
    w.st.cap = cap;
    w.st.j = c.take<int32_t>(cap > 0 ? cap : 1);
    w.st.udf = c.take<double>(cap > 0 ? cap : 1);
    w.st.alpha = c.take<double>(cap > 0 ? cap : 1);
    w.st.w = c.take<double>(cap > 0 ? cap : 1);
    w.st.col = color ? c.take<double>(3 * (cap > 0 ? cap : 1)) : nullptr;
    w.gds = big ? c.take<double>(kSampleGrid * max_q) : nullptr;
    w.gidx = big ? c.take<int>(kSampleGrid * max_q) : nullptr;
    w.scan = c.take<char>(scan_workspace_bytes(m + 1));
    return w;
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

Params to_params(const hp_sampler_params* p) {
    Params P;
    P.K = p->k_neighbors;
    P.eps_mode = p->eps_mode;
    P.want_color = p->want_color;
    P.exact_t_end = p->exact_t_end;
    P.beta2 = p->beta2;
    P.gamma = p->gamma;
    P.eps = p->eps;
    P.tau_min = p->tau_min;
    return P;
}

template <class BestT>
int launch_sample(const Csr& C, const Params& P, int mode, const int* list, const int* list_n, const SampleWs& w,
                  int64_t* rcount, double* t_end, const int64_t* r_off, const Outputs& O, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_sample<BestT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(RaySmem)));
        attr = true;
    }
    k_sample<BestT><<<kSampleGrid, kThreads, sizeof(RaySmem), s>>>(C, P, mode, list, list_n, w.gds, w.gidx, rcount,
                                                               t_end, w.ray_stage, w.stage_cursor, w.st,
                                                               w.ovf_list, w.ovf_n, r_off, O);
    HP_CHECK_LAUNCH("k_sample");
    return HP_OK;
}

int dispatch_sample(const Csr& C, const Params& P, int mode, const int* list, const int* list_n, const SampleWs& w,
                    int64_t* rcount, double* t_end, const int64_t* r_off, const Outputs& O, cudaStream_t s) {
    if (P.K <= 8) return launch_sample<Best<8>>(C, P, mode, list, list_n, w, rcount, t_end, r_off, O, s);
    if (P.K <= 32) return launch_sample<Best<32>>(C, P, mode, list, list_n, w, rcount, t_end, r_off, O, s);
    return launch_sample<BestDyn>(C, P, mode, list, list_n, w, rcount, t_end, r_off, O, s);
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


extern "C" int hp_sample_workspace_bytes(int64_t m, int64_t total, int64_t max_q, int64_t stage_capacity,
                                         const hp_sampler_params* p, size_t* bytes) {
    Carver c(nullptr, 0);
    // the global scratch for long rays is sized by `total` and only exists
    // when some ray has more than kSmemCap candidates
    carve_sample(c, m, total, stage_capacity, p && p->want_color, max_q);
    *bytes = c.used + 256;
    return HP_OK;
}

extern "C" int hp_sample_run(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                             const double* dist, int64_t total, int64_t max_q, const double* slopes,
                             const hp_sampler_params* p, const double* colors, int64_t n_colors,
                             int64_t stage_capacity, int64_t* r_off, double* t_end, void* workspace,
                             size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, total, stage_capacity, p->want_color, max_q);
    if (!c.ok()) {
        set_error("hp_sample_run: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(w.stage_cursor, 0, sizeof(int64_t), s) != cudaSuccess ||
        cudaMemsetAsync(w.ovf_n, 0, sizeof(int), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_sample_run memset");
    Csr C{offsets, ids, t, dist, slopes, colors, m, max_q};
    Params P = to_params(p);
    Outputs O{};
    if (m > 0) HP_TRY(dispatch_sample(C, P, 0, nullptr, nullptr, w, r_off, t_end, nullptr, O, s));
    HP_TRY(exclusive_scan_i64(r_off, r_off, m, w.scan, s));
    return HP_OK;
}

extern "C" int hp_sample_emit(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                              const double* dist, int64_t total, int64_t max_q, const double* slopes,
                              const hp_sampler_params* p, const double* colors, int64_t n_colors,
                              int64_t stage_capacity, const int64_t* r_off, int64_t R, int64_t* r_id, double* r_t,
                              double* r_dist, double* r_udf, double* r_alpha, double* r_w, double* r_color,
                              void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    HP_TRY(validate(p, colors, n_colors));
    if (R == 0 || m == 0) return HP_OK;
    Carver c(workspace, workspace_bytes);
    SampleWs w = carve_sample(c, m, total, stage_capacity, p->want_color, max_q);
    if (!c.ok()) {
        set_error("hp_sample_emit: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Csr C{offsets, ids, t, dist, slopes, colors, m, max_q};
    Params P = to_params(p);
    Outputs O{r_id, r_t, r_dist, r_udf, r_alpha, r_w, r_color};
    k_emit<<<grid_for(m * 32, 256), 256, 0, s>>>(C, P, r_off, w.ray_stage, w.st, O);
    HP_CHECK_LAUNCH("k_emit");
    // rays whose retained list overflowed the staging: recompute, write direct
    HP_TRY(dispatch_sample(C, P, 1, w.ovf_list, w.ovf_n, w, nullptr, nullptr, r_off, O, s));
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
    if (cudaMemcpyFromSymbol(h, g_dbg, sizeof(h)) != cudaSuccess) return cuda_status(cudaGetLastError(), "dbg");
    for (int k = 0; k < 8; k++) out8[k] = int64_t(h[k]);
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
    }
    return HP_OK;
}
