// hp_sample_core.cuh — the sampler's per-candidate arithmetic (K-nearest
// search, udf / alpha / colour, bound factors, bound chain) used by the
// sampler kernels in hp_sample.cu.  Reference: _kernels.sample_batch
// (_kernels.py:552-700); exactness arguments in DESIGN.md §6.
#pragma once
#include <math_constants.h>

#include <cfloat>
#include <climits>
#include <cmath>

#include "hp_common.cuh"

// the exact sampler's K-nearest walk: seed window, then each side alone (1),
// or one merged two-sided walk (0); DESIGN.md §5 "Sampler"
#ifndef HP_EXACT_SIDES
#define HP_EXACT_SIDES 1
#endif
#ifndef HP_EXACT_SEED
#define HP_EXACT_SEED 4
#endif
#ifndef HP_EXACT_LA
#define HP_EXACT_LA 1
#endif
#ifndef HP_EXACT_SORTSEED
#define HP_EXACT_SORTSEED 1
#endif

namespace hp {
namespace {

struct Params {
    int K;
    int eps_mode, want_color, exact_t_end, emit_knn;
    double beta2, gamma, eps, tau_min;
    double inv_beta2_up;  // 1 / beta2 rounded up (bound factors only)
    double inv_k_up;      // 1 / K rounded up (bound factors only)
    float inv_beta2_up_f;  // the same two, as floats rounded up (fp32 bound factors)
    float inv_k_up_f;
    int f32_bounds;        // the fp32 ring bound is usable (inv_beta2_up_f finite)
};

__device__ __forceinline__ bool kless(double d2a, int ia, double d2b, int ib) {
    return d2a < d2b || (d2a == d2b && ia < ib);
}

// K-best list in registers (MAXK compile-time, ksel <= MAXK at runtime),
// ascending by (d2, i).
template <int MAXK>
struct Best {
    static constexpr int kMax = MAXK;
    double d[MAXK];
    int i[MAXK];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int b = 0; b < MAXK; b++) {
            d[b] = CUDART_INF;
            i[b] = INT_MAX;
        }
    }
    // d[ksel - 1] as a select chain: an equality test lets the compiler turn
    // the loop into one indexed load, which demotes the list to local memory.
    __device__ __forceinline__ void kth(int ksel, double& kd, int& ki) const {
        double x = d[0];
        int y = i[0];
#pragma unroll
        for (int b = 1; b < MAXK; b++) {
            const bool in = b < ksel;
            x = in ? d[b] : x;
            y = in ? i[b] : y;
        }
        kd = x;
        ki = y;
    }
    template <class F>
    __device__ __forceinline__ void for_each(int ksel, F f) const {
#pragma unroll
        for (int b = 0; b < MAXK; b++)
            if (b < ksel) f(d[b], i[b]);
    }
    // full list (ksel == MAXK): branch-free compare-shift network; the caller
    // guarantees (nd, ni) < the last entry.  One comparison per slot: keys
    // are unique (ids differ) and the list is sorted, so lt[b] = (entry b <
    // new) is true exactly below the insertion point.
    __device__ __forceinline__ void insert_full(double nd, int ni) {
        bool lt[MAXK];
#pragma unroll
        for (int b = 0; b < MAXK; b++) lt[b] = kless(d[b], i[b], nd, ni);
#pragma unroll
        for (int b = MAXK - 1; b >= 1; --b) {
            const bool shift = !lt[b - 1];
            const bool here = lt[b - 1] && !lt[b];
            d[b] = shift ? d[b - 1] : (here ? nd : d[b]);
            i[b] = shift ? i[b - 1] : (here ? ni : i[b]);
        }
        if (!lt[0]) {
            d[0] = nd;
            i[0] = ni;
        }
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
    static constexpr int kMax = HP_MAX_K;
    double d[HP_MAX_K];
    int i[HP_MAX_K];
    __device__ void init() {
        for (int b = 0; b < HP_MAX_K; b++) {
            d[b] = CUDART_INF;
            i[b] = INT_MAX;
        }
    }
    __device__ void kth(int ksel, double& kd, int& ki) const {
        kd = d[ksel - 1];
        ki = i[ksel - 1];
    }
    template <class F>
    __device__ void for_each(int ksel, F f) const {
        for (int b = 0; b < ksel; b++) f(d[b], i[b]);
    }
    __device__ void insert_full(double nd, int ni) { insert(HP_MAX_K, nd, ni); }
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

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// One ray's t / ds segment of the query CSR (read-only path).
struct RayView {
    const double* gt;
    const double* gd;
    __device__ __forceinline__ double t(int i) const { return __ldg(gt + i); }
    __device__ __forceinline__ double d(int i) const { return __ldg(gd + i); }
};

// Exact udf/alpha (and colour) of candidate j (reference _kernels.py:594-660).
// q candidates are present of the ray's qt (prefix mode: q < qt, the others
// all at t >= tcut, fast path only).  Returns false when the K nearest may
// lie past the prefix (the ray then takes the full path).
template <class BestT, class View, class IdT>
__device__ bool eval_exact(const View& V, int q, int qt, double tcut, int j, bool fast,
                           int jstar, double slope, const Params& P, const IdT* __restrict__ ids_ray,
                           const double* __restrict__ colors, double& udf, double& alpha, double* col3,
                           unsigned long long& evals, int64_t* knn_id = nullptr, double* knn_w = nullptr) {
    const double tj = V.t(j);
    const double rj = dmul(slope, tj);
    const bool partial = q < qt;
    bool use_el;
    int ksel;
    if (fast) {
        use_el = j >= jstar;
        ksel = use_el ? P.K : (qt < P.K ? qt : P.K);
    } else {
        int n_el = 0;
        for (int i = 0; i < q; i++) n_el += (V.d(i) <= rj);
        use_el = n_el >= P.K;
        const int pool = use_el ? n_el : q;
        ksel = pool > P.K ? P.K : pool;
    }
    BestT best;
    best.init();
    double kd = CUDART_INF;
    int ki = INT_MAX;
    constexpr int kMaxK = BestT::kMax;
    const bool full = ksel == kMaxK;
    // one pool member i at (t_i, ds_i): returns false once (t_i - t_j)^2
    // exceeds the K-th best (every point further out on that side is then out)
    auto visit = [&](int i, double ti, double di) -> bool {
        const double dt = dsub(ti, tj);
        const double lb = dmul(dt, dt);
        if (lb > kd) return false;
        if (use_el && di > rj) return true;
        const double d2 = dadd(lb, dmul(di, di));
        evals++;
        if (kless(d2, i, kd, ki)) {
            if (full) {
                best.insert_full(d2, i);
                kd = best.d[kMaxK - 1];
                ki = best.i[kMaxK - 1];
            } else if (kMaxK <= 8) {
                best.insert_full(d2, i);
                best.kth(ksel, kd, ki);
            } else {
                best.insert(ksel, d2, i);
                best.kth(ksel, kd, ki);
            }
        }
        return true;
    };
#if HP_EXACT_SIDES
    if (fast) {
        // The K nearest do not depend on the visiting order: a side is left
        // only at a point with (t_i - t_j)^2 > the current K-th best >= the
        // final one, and every point further out on that side is at least as
        // far in t.  So: a seed window j - kSeed .. j + kSeed (a tight bound
        // of the K-th best), then each side outward with its own simple loop
        // (the next point loaded one step ahead).  Prefix mode: when the right
        // side runs out of the prefix, the cut is a lower bound of the t of
        // every left-out match.
        constexpr int kSeed = HP_EXACT_SEED;
        const int s0 = j - kSeed > 0 ? j - kSeed : 0;
        const int s1 = j + kSeed + 1 < q ? j + kSeed + 1 : q;
#if HP_EXACT_SORTSEED
        if constexpr (kMaxK == 8 && kSeed == 4) {
            // the 9 seed points sorted by one network (25 compare-exchanges,
            // checked by the 0-1 principle) instead of 9 insertions: the 8
            // smallest of the 9 in (d2, i) order are exactly what the
            // insertions leave; missing / out-of-pool points are (inf, INT_MAX)
            double sd[9];
            int si[9];
#pragma unroll
            for (int b = 0; b < 9; b++) {
                const int i = j - kSeed + b;
                sd[b] = CUDART_INF;
                si[b] = INT_MAX;
                if (i >= s0 && i < s1) {
                    const double ti = V.t(i), di = V.d(i);
                    if (!(use_el && di > rj)) {
                        const double dt = dsub(ti, tj);
                        sd[b] = dadd(dmul(dt, dt), dmul(di, di));
                        si[b] = i;
                        evals++;
                    }
                }
            }
            constexpr int kNet[25][2] = {{0, 1}, {3, 4}, {6, 7}, {1, 2}, {4, 5}, {7, 8}, {0, 1}, {3, 4}, {6, 7},
                                         {0, 3}, {3, 6}, {0, 3}, {1, 4}, {4, 7}, {1, 4}, {2, 5}, {5, 8}, {2, 5},
                                         {1, 3}, {5, 7}, {2, 6}, {4, 6}, {2, 4}, {2, 3}, {5, 6}};
#pragma unroll
            for (int c = 0; c < 25; c++) {
                const int a = kNet[c][0], b = kNet[c][1];
                const bool sw = kless(sd[b], si[b], sd[a], si[a]);
                const double da = sw ? sd[b] : sd[a], db = sw ? sd[a] : sd[b];
                const int ia = sw ? si[b] : si[a], ib = sw ? si[a] : si[b];
                sd[a] = da;
                sd[b] = db;
                si[a] = ia;
                si[b] = ib;
            }
#pragma unroll
            for (int b = 0; b < 8; b++) {
                best.d[b] = sd[b];
                best.i[b] = si[b];
            }
            best.kth(ksel, kd, ki);
        } else
#endif
        for (int i = s0; i < s1; i++) visit(i, V.t(i), V.d(i));
#if HP_EXACT_LA == 2
        if (s0 > 0) {
            double tn = V.t(s0 - 1), dn = V.d(s0 - 1);
            const int n2 = s0 > 1 ? s0 - 2 : 0;
            double tm = V.t(n2), dm = V.d(n2);
            for (int i = s0 - 1; i >= 0; --i) {
                const double ti = tn, di = dn;
                tn = tm;
                dn = dm;
                const int nx = i > 1 ? i - 2 : 0;
                tm = V.t(nx);
                dm = V.d(nx);
                if (!visit(i, ti, di)) break;
            }
        }
        int r = s1;
        if (r < q) {
            double tn = V.t(r), dn = V.d(r);
            const int n2 = r + 1 < q ? r + 1 : r;
            double tm = V.t(n2), dm = V.d(n2);
            for (; r < q; ++r) {
                const double ti = tn, di = dn;
                tn = tm;
                dn = dm;
                const int nx = r + 2 < q ? r + 2 : q - 1;
                tm = V.t(nx);
                dm = V.d(nx);
                if (!visit(r, ti, di)) break;
            }
        }
#else
        if (s0 > 0) {
            double tn = V.t(s0 - 1), dn = V.d(s0 - 1);
            for (int i = s0 - 1; i >= 0; --i) {
                const double ti = tn, di = dn;
                const int nx = i > 0 ? i - 1 : 0;
                tn = V.t(nx);
                dn = V.d(nx);
                if (!visit(i, ti, di)) break;
            }
        }
        int r = s1;
        if (r < q) {
            double tn = V.t(r), dn = V.d(r);
            for (; r < q; ++r) {
                const double ti = tn, di = dn;
                const int nx = r + 1 < q ? r + 1 : r;
                tn = V.t(nx);
                dn = V.d(nx);
                if (!visit(r, ti, di)) break;
            }
        }
#endif
        if (partial && r == q) {
            const double dc = dsub(tcut, tj);
            if (!(dmul(dc, dc) > kd)) return false;
        }
    } else
#endif
    if (fast) {
        // outward from j in t order; stop once (t_i - t_j)^2 > K-th best
        // (t, ds) of the next candidate on each side are loaded one step ahead
        // prefix mode: past the prefix, the cut stands in for the next
        // candidate on the right (a lower bound of its t)
        int l = j, r = j + 1;
        const int rend = partial ? q + 1 : q;
        double tl = tj, dl = V.d(j), tr = tcut, dr = 0.0;
        if (r < q) {
            tr = V.t(r);
            dr = V.d(r);
        }
        while (l >= 0 || r < rend) {
            const bool go_left = l >= 0 && (r >= rend || dsub(tj, tl) <= dsub(tr, tj));
            int i;
            double ti, di;
            if (go_left) {
                i = l;
                ti = tl;
                di = dl;
                if (--l >= 0) {
                    tl = V.t(l);
                    dl = V.d(l);
                }
            } else {
                if (r == q) {  // the cut: every left-out match is at least this far
                    const double dc = dsub(tcut, tj);
                    if (dmul(dc, dc) > kd) break;
                    return false;
                }
                i = r;
                ti = tr;
                di = dr;
                if (++r < q) {
                    tr = V.t(r);
                    dr = V.d(r);
                } else {
                    tr = tcut;
                }
            }
            const double dt = dsub(ti, tj);
            const double lb = dmul(dt, dt);
            if (lb > kd) break;  // the other side is at least as far
            if (use_el && di > rj) continue;
            const double d2 = dadd(lb, dmul(di, di));
            evals++;
            if (kless(d2, i, kd, ki)) {
                if (full) {
                    best.insert_full(d2, i);
                    kd = best.d[kMaxK - 1];
                    ki = best.i[kMaxK - 1];
                } else if (kMaxK <= 8) {
                    // small register list: the branch-free network over all
                    // slots (what it pushes past slot ksel - 1 is never read)
                    best.insert_full(d2, i);
                    best.kth(ksel, kd, ki);
                } else {
                    best.insert(ksel, d2, i);
                    best.kth(ksel, kd, ki);
                }
            }
        }
    } else {
        for (int i = 0; i < q; i++) {  // reference loop (_kernels.py:607-620)
            const double di = V.d(i);
            if (use_el && di > rj) continue;
            const double dt = dsub(V.t(i), tj);
            const double d2 = dadd(dmul(dt, dt), dmul(di, di));
            evals++;
            if (d2 < kd) {
                best.insert(ksel, d2, i);
                best.kth(ksel, kd, ki);
            }
        }
    }
    double acc = 0.0;
    best.for_each(ksel, [&](double d2, int) { acc = dadd(acc, sqrt(d2)); });
    udf = __ddiv_rn(acc, double(ksel));
    alpha = dmul(P.gamma, exp(__ddiv_rn(-dmul(udf, udf), P.beta2)));
    if (knn_id) {  // the K nearest's point ids and blend weights (the colour blend's)
        int nz = 0;
        double wsum = 0.0;
        best.for_each(ksel, [&](double d2, int) { nz += (d2 == 0.0); });
        if (nz == 0) best.for_each(ksel, [&](double d2, int) { wsum = dadd(wsum, __ddiv_rn(1.0, sqrt(d2))); });
        int b = 0;
        best.for_each(ksel, [&](double d2, int i) {
            knn_id[b] = int64_t(ids_ray[i]);
            knn_w[b] = nz > 0 ? (d2 == 0.0 ? __ddiv_rn(1.0, double(nz)) : 0.0)
                              : __ddiv_rn(__ddiv_rn(1.0, sqrt(d2)), wsum);
            b++;
        });
        for (; b < P.K; b++) {
            knn_id[b] = -1;
            knn_w[b] = 0.0;
        }
    }
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
    return true;
}

// Upper bound of the reference's factor fl(1 - alpha_j) (DESIGN.md "sampler:
// transmittance bound").  For any ksel members A of j's pool,
//   sum_{K nearest} sqrt(d2) <= sum_A sqrt(dt^2 + ds^2) <= sum_A (|dt| + ds),
// so the mean of (|dt| + ds) over the first ksel pool members at or after j
// in t order (then before j) bounds udf_j from above once inflated by 1e-12
// (which dominates every fp64 rounding of both sums for K <= 256).  exp is
// then bounded below in fp32 (argument rounded up, result scaled by
// 1 - 2^-20 against expf's 2-ulp error).  Every later operation is monotone,
// so U_{j+1} = U_j * u_j in the reference's order dominates T_j.
__device__ __forceinline__ double factor_from_sum(double sum, int ksel, const Params& P) {
    // x / ksel bounded above without a division: RU(x * RU(1 / ksel)) >= x / ksel
    const double inv_up = ksel == P.K ? P.inv_k_up : __drcp_ru(double(ksel));
    const double udf_up = __dmul_ru(dmul(sum, 1.0 + 1e-12), inv_up);
    const double y = dmul(dmul(udf_up, udf_up), P.inv_beta2_up);  // >= fl(udf^2) / beta^2
    const float e = expf(-__double2float_ru(y));
    const double a_lo = dmul(P.gamma, dmul(double(e), 1.0 - 0x1p-20));
    return dsub(1.0, a_lo);
}

// The same bound in fp32 with directed rounding (half the fp64 pipe work of
// factor_from_sum): sum >= the exact real sum of (|dt| + ds) over the ksel
// members; the 2^-20 inflation dominates every fp64 rounding of the
// reference's udf (K <= 256), and y >= the reference's exp argument.
__device__ __forceinline__ double factor_from_sum_f(float sum, int ksel, const Params& P) {
    const float inv_up = ksel == P.K ? P.inv_k_up_f : __frcp_ru(float(ksel));
    const float udf_up = __fmul_ru(__fmul_ru(sum, 1.0f + 0x1p-20f), inv_up);
    const float y = __fmul_ru(__fmul_ru(udf_up, udf_up), P.inv_beta2_up_f);
    const float e = expf(-y);
    const double a_lo = dmul(P.gamma, dmul(double(e), 1.0 - 0x1p-20));
    return dsub(1.0, a_lo);
}

template <class View>
__device__ double bound_factor(const View& V, int q, int j, int jstar, double slope, const Params& P) {
    const double tj = V.t(j);
    const double rj = dmul(slope, tj);
    const bool use_el = j >= jstar;
    const int ksel = use_el ? P.K : (q < P.K ? q : P.K);
    double sum = 0.0;
    int found = 0;
    for (int i = j; i < q && found < ksel; i++) {
        const double di = V.d(i);
        if (use_el && di > rj) continue;
        sum = dadd(sum, dadd(dsub(V.t(i), tj), di));
        found++;
    }
    for (int i = j - 1; found < ksel; i--) {  // the pool has >= ksel members
        const double di = V.d(i);
        if (use_el && di > rj) continue;
        sum = dadd(sum, dadd(dsub(tj, V.t(i)), di));
        found++;
    }
    return factor_from_sum(sum, ksel, P);
}

// Same bound with the members taken from the warp's ring of the last 64
// candidates (K <= 32): the ksel candidates ending at j (or [0, ksel) for
// j < ksel - 1).  Returns a negative value when a member is not in j's pool
// (the caller then uses bound_factor).
template <int kRingSize>
__device__ __forceinline__ double bound_factor_ring(const double* rt, const double* rd, int q, int j, double tj,
                                                    int jstar, double slope, const Params& P) {
    const bool use_el = j >= jstar;
    const int ksel = use_el ? P.K : (q < P.K ? q : P.K);
    const double rj = dmul(slope, tj);
    const int i0 = j >= ksel - 1 ? j - ksel + 1 : 0;
    double sum = 0.0;
    bool ok = true;
    for (int k = 0; k < ksel; k++) {
        const int i = (i0 + k) & (kRingSize - 1);
        const double di = rd[i];
        ok &= !(use_el && di > rj);
        sum = dadd(sum, dadd(fabs(dsub(rt[i], tj)), di));
    }
    return ok ? factor_from_sum(sum, ksel, P) : -1.0;
}

// fp32 ring variant for j >= ksel - 1 (members [j - ksel + 1, j], all at or
// before j).  rf[i] = (RD(t_i - tb), RU(ds_i)) for the ray's base tb,
// thi = RU(t_j - tb), rj_lo = RD(slope * t_j): thi - rf[i].x >= t_j - t_i and
// rf[i].y <= rj_lo proves ds_i <= r_j.  Negative: a member may be outside the
// pool (the caller then uses bound_factor).
template <int kRingSize>
__device__ __forceinline__ double bound_factor_ringf(const float2* rf, int j, float thi, float rj_lo, int ksel,
                                                     bool use_el, const Params& P) {
    float sum = 0.0f;
    bool ok = true;
    if (ksel == 8) {  // the default K: unrolled
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const float2 e = rf[(j - k) & (kRingSize - 1)];
            ok &= !(use_el && e.y > rj_lo);
            sum = __fadd_ru(sum, __fadd_ru(__fsub_ru(thi, e.x), e.y));
        }
    } else {
        for (int k = 0; k < ksel; k++) {
            const float2 e = rf[(j - k) & (kRingSize - 1)];
            ok &= !(use_el && e.y > rj_lo);
            sum = __fadd_ru(sum, __fadd_ru(__fsub_ru(thi, e.x), e.y));
        }
    }
    return ok ? factor_from_sum_f(sum, ksel, P) : -1.0;
}

// Warp: first j in [0, q) with pred(j) (monotone false..true); q if none.
template <class Pred>
__device__ int warp_first_true(int q, Pred pred) {
    int a = 0, b = q;  // answer in [a, b]
    const int lane = lane_id();
    while (b - a > 32) {
        const int stride = (b - a + 31) / 32;
        const int j = a + lane * stride;
        const bool p = j < b && pred(j);
        const unsigned mask = __ballot_sync(0xffffffffu, p);
        const unsigned valid = __ballot_sync(0xffffffffu, j < b);
        if (mask == 0) {
            a = a + (31 - __clz(valid)) * stride + 1;
        } else {
            const int f = __ffs(mask) - 1;
            b = a + f * stride;
            if (f > 0) a = a + (f - 1) * stride + 1;
        }
    }
    const int j = a + lane;
    const unsigned mask = __ballot_sync(0xffffffffu, j < b && pred(j));
    return mask ? a + __ffs(mask) - 1 : b;
}


// ---- bound chain (DESIGN.md §6 "Early exit with an exact transmittance").
// Vs bounds the reference's T at the current chunk start.  While it is far
// from underflow, the chunk's bounds come from a round-up warp prefix
// product: T_{c0+l+1} <= T_{c0} * prod f * (1+u)^(l+1) + (l+1) 2^-1075
// (round-to-nearest error <= u|x| + 2^-1075 per step), and prod f <= prod u
// (round-up).  Near underflow the sequential round-to-nearest chain
// U_{i+1} = U_i * u_i (monotone, dominates T_i) takes over and proves the
// exact zero.  je: retention is decided before je.
struct Chain {
    double Vs = 1.0;
    bool seq = false;
    int je = 0;
    bool proved_zero = false;
};

// Warp-uniform step over the bound factors u (one per lane, 1.0 beyond the
// ray) of candidates [c0, c0 + n).  Returns true when the chain is finished.
__device__ __forceinline__ bool chain_chunk(Chain& S, double u, int c0, int n, int q, double thr, const Params& P) {
    const int lane = lane_id();
    if (!S.seq) {
        // Tail proof without the sequential chain: below 2^-1022 the
        // reference's T is n units of 2^-1074, and a factor <= 1/2 maps n to
        // at most ceil(n / 2) (round to nearest even; 1 -> 0).  From T <= Vs <=
        // 2^-1049 (n <= 2^25), 26 factors <= 1/2 reach exactly 0.
        if (S.Vs <= 0x1p-1049 && S.je < q && n >= 26 &&
            __all_sync(0xffffffffu, lane >= n || u <= 0.5)) {
            S.proved_zero = true;
            return true;
        }
        double Pl = u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double other = __shfl_up_sync(0xffffffffu, Pl, o);
            if (lane >= o) Pl = __dmul_ru(Pl, other);
        }
        double B = __dmul_ru(__dmul_ru(S.Vs, Pl), 1.0 + double(lane + 1) * 0x1p-51);
        B = __dadd_ru(B, double(lane + 1) * 0x1p-1074);
        if (S.je == q) {
            if (S.Vs < thr) {
                S.je = c0;
            } else {
                const unsigned mask = __ballot_sync(0xffffffffu, lane < n && B < thr);
                if (mask) S.je = c0 + __ffs(mask);  // T_{c0+l+1} < thr for the first such l
            }
        }
        const double Vn = __shfl_sync(0xffffffffu, B, n - 1);
        if (Vn >= 0x1p-1000 || (S.Vs >= 0x1p-1000 && S.je < q)) {
            // far from underflow; or the first chunk below it: its end bound
            // may open the tail proof above for the next chunk
            S.Vs = Vn;
            return !P.exact_t_end && S.je < q;
        }
        S.seq = true;  // redo this chunk sequentially from Vs
    }
    double U = S.Vs;
    for (int k = 0; k < n; k++) {
        const double uk = __shfl_sync(0xffffffffu, u, k);
        if (S.je == q && U < thr) S.je = c0 + k;
        U = dmul(U, uk);
        if (U == 0.0) {
            S.proved_zero = true;
            if (S.je == q && thr > 0.0) S.je = c0 + k + 1;  // U_{j+1} = 0 < thr
            break;
        }
    }
    S.Vs = U;
    return S.proved_zero || (!P.exact_t_end && S.je < q);
}

}  // namespace
}  // namespace hp
