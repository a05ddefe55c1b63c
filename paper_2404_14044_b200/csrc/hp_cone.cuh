// hp_cone.cuh — the per-(ray, point) cone test: the reference's fp64 test and
// the float32 filter in front of it.  __host__ __device__ so that
// tests/cone_filter_check.cu can stress the filter's soundness on the CPU.
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define HP_HD __host__ __device__ __forceinline__
#else
#define HP_HD inline
#endif

namespace hp {

// Without FMA contraction (the library is compiled with -fmad=false; on the
// host the test compiles with -ffp-contract=off): IEEE round-to-nearest ops.
HP_HD double cmul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
HP_HD double cadd(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
HP_HD double csub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}

struct RayParams {
    int u, v;  // padded window origin (== unpadded pixel)
    double d0, d1, d2, tn, tf, slope;
    float f0, f1, f2, ftn, ftf, fslope, eps_ray, smax;
};

// _cone_test (_kernels.py:22-36): t = p.d; reject outside [tn, tf]; reject
// when |p - t d|^2 > (t * slope)^2.  Returns the exact fp64 t and dist^2.
// t = p.d and |p - t d|^2 in the reference's operation order (no FMA); the
// query sort recomputes dist^2 from the same p, t and d (bit-identical).
HP_HD double cone_t(double p0, double p1, double p2, double d0, double d1, double d2) {
    return cadd(cadd(cmul(p0, d0), cmul(p1, d1)), cmul(p2, d2));
}
HP_HD double cone_dist2(double p0, double p1, double p2, double t, double d0, double d1, double d2) {
    const double e0 = csub(p0, cmul(t, d0));
    const double e1 = csub(p1, cmul(t, d1));
    const double e2 = csub(p2, cmul(t, d2));
    return cadd(cadd(cmul(e0, e0), cmul(e1, e1)), cmul(e2, e2));
}

HP_HD bool cone_test(double p0, double p1, double p2, const RayParams& r,
                                          double& t, double& dist2) {
    t = cone_t(p0, p1, p2, r.d0, r.d1, r.d2);
    if (t < r.tn || t > r.tf) return false;
    dist2 = cone_dist2(p0, p1, p2, t, r.d0, r.d1, r.d2);
    const double rad = cmul(t, r.slope);
    return !(dist2 > cmul(rad, rad));
}

// float32 filter.  P = (x, y, z, e) with e = 2^-18 |p|_1 (rounded up).  The
// band eps = e * max(1, slope) + 2^-22 * t_far bounds |t32 - t64| and the
// error of the fp32 perpendicular distance (derivation in DESIGN.md).
// Returns 0 = reject, 1 = accept, 2 = decide in fp64.
// The filter's float terms of a ray (held in registers across a run of slots).
struct RayF {
    float f0, f1, f2, ftn, ftf, fslope, eps_ray, smax;
};
HP_HD RayF ray_f(const RayParams& r) { return RayF{r.f0, r.f1, r.f2, r.ftn, r.ftf, r.fslope, r.eps_ray, r.smax}; }

// cone_filter that also hands back the float t and band eps: for an accepted
// pair |t - t64| <= eps (the band covers the t error bound with a wide
// margin), so t - eps rounded down is a lower bound of the exact t.
HP_HD int cone_filter_te(const float4 P, const RayF& r, float& t, float& eps) {
    // every term computed, the decision by selects (no early exits: the warp
    // runs all paths anyway, and branch-free code schedules better)
    eps = fmaf(P.w, r.smax, r.eps_ray);
    t = fmaf(P.z, r.f2, fmaf(P.y, r.f1, P.x * r.f0));
    const bool t_out = t < r.ftn - eps || t > r.ftf + eps;
    const float ex = fmaf(-t, r.f0, P.x), ey = fmaf(-t, r.f1, P.y), ez = fmaf(-t, r.f2, P.z);
    const float d2 = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
    const float rr = t * r.fslope;
    const float hi = rr + eps;
    const bool d_out = d2 > hi * hi * (1.0f + 0x1p-20f);
    const float lo = rr - eps;
    const bool t_in = (t >= r.ftn + eps) && (t <= r.ftf - eps);
    const bool sure = t_in && lo > 0.0f && d2 < lo * lo * (1.0f - 0x1p-20f);
    return (t_out || d_out) ? 0 : (sure ? 1 : 2);
}
HP_HD int cone_filter(const float4 P, const RayF& r) {
    float t, eps;
    return cone_filter_te(P, r, t, eps);
}
HP_HD int cone_filter(const float4 P, const RayParams& r) { return cone_filter(P, ray_f(r)); }


// Ray parameters derived once per ray (float copies, filter band terms).
HP_HD void ray_derive(RayParams& p) {
    p.f0 = float(p.d0);
    p.f1 = float(p.d1);
    p.f2 = float(p.d2);
    p.ftn = float(p.tn);
    p.ftf = float(p.tf);
    p.fslope = float(p.slope);
    const float tmax = fmaxf(fabsf(p.ftn), fabsf(p.ftf));
    p.eps_ray = (tmax <= 3.402823466e38f) ? tmax * 0x1p-22f : INFINITY;
    p.smax = fmaxf(1.0f, fabsf(p.fslope));
    if (!(p.smax <= 3.402823466e38f)) p.smax = INFINITY;
}

// float32 copy of an origin-relative point with its error budget
// e = 2^-18 * |p|_1, rounded up.
HP_HD float4 filter_point(double x, double y, double z) {
    const float fx = float(x), fy = float(y), fz = float(z);
    const double l1 = (double(fabsf(fx)) + double(fabsf(fy))) + double(fabsf(fz));
    float e = float(l1 * 0x1p-18 * (1.0 + 0x1p-20));
    if (double(e) < l1 * 0x1p-18) e = nextafterf(e, INFINITY);
    return make_float4(fx, fy, fz, e);
}

// ------------------------------------------------------------------ footprint
// Which pixels of a ray's s x s window can hold an accepted point.  The cone
// test accepts p iff t = p.d > 0 and |p - t d| <= slope * t, i.e. iff the
// angle between p and d is at most atan(slope).  A point's pixel depends only
// on its direction (U = f (p.R)/(p.F)/pw + W/2, V = -f (p.U)/(p.F)/ph + H/2),
// and the directions within that angle project to an ellipse on the image
// plane (when the cone does not reach the image plane's horizon).  Per padded
// row y the accepted points therefore lie in a column interval, computed here
// with margins: the half-angle widened by 1e-7 relative (covers the fp64 test's
// rounding), the row slab widened by 1e-3 pixel (covers rounding of V in the
// build), one extra column on each side (rounding of U).  tests/native/
// footprint_check.cu verifies the bound against the reference cone test.
struct CamFrame {
    double r[3], u[3], f[3];
    double focal, pw, ph, half_w, half_h;
};

struct Footprint {
    int tight;  // 0: use the full window
    double dx, dy, dz, c2, amin, amax, bL, bR, bmin, bmax;
};

// Roots of A x^2 + 2 B x + C = 0 (A != 0), sorted; false when complex.
HP_HD bool roots2(double A, double B, double C, double& x0, double& x1) {
    double disc = B * B - A * C;
    if (!(disc >= 0.0)) return false;
    const double sq = sqrt(disc);
    const double r0 = (-B + sq) / A, r1 = (-B - sq) / A;
    x0 = fmin(r0, r1);
    x1 = fmax(r0, r1);
    return true;
}

HP_HD void footprint_init(Footprint& F, const CamFrame& C, double d0, double d1, double d2, double slope) {
    F.tight = 0;
    F.dx = d0 * C.r[0] + d1 * C.r[1] + d2 * C.r[2];
    F.dy = d0 * C.u[0] + d1 * C.u[1] + d2 * C.u[2];
    F.dz = d0 * C.f[0] + d1 * C.f[1] + d2 * C.f[2];
    const double sig = slope * (1.0 + 1e-7) + 1e-12;
    if (!(sig >= 0.0) || !(sig < 1e3)) return;
    F.c2 = 1.0 / (1.0 + sig * sig);
    const double s2 = sig * sig * F.c2;
    const double dz = F.dz, dx = F.dx, dy = F.dy, f = C.focal;
    // bounded ellipse with margin: the cone edge at least ~0.6 degree from the horizon
    if (!(dz > 0.0) || !(dz * dz - s2 > 1e-4)) return;
    const double A2 = s2 - dz * dz;  // < 0
    const double k = F.c2 - dy * dy, kp = F.c2 - dx * dx;
    if (!(k > 0.0) || !(kp > 0.0)) return;
    if (!roots2(A2, dx * f * dz, f * f * (dz * dz - k), F.amin, F.amax)) return;
    if (!roots2(A2, dy * f * dz, f * f * (dz * dz - kp), F.bmin, F.bmax)) return;
    F.bL = dy * (F.amin * dx + f * dz) / k;
    F.bR = dy * (F.amax * dx + f * dz) / k;
    F.tight = 1;
}

// a-interval of the ellipse at height b (empty if outside).
HP_HD void footprint_a_at(const Footprint& F, const CamFrame& C, double b, double& lo, double& hi) {
    const double A = F.dx * F.dx - F.c2;  // < 0 when tight
    const double w = b * F.dy + C.focal * F.dz;
    const double B = F.dx * w;
    const double Cq = w * w - F.c2 * (b * b + C.focal * C.focal);
    double disc = B * B - A * Cq;
    if (disc < 0.0) disc = 0.0;  // tangency up to rounding
    const double sq = sqrt(disc);
    const double r0 = (-B + sq) / A, r1 = (-B - sq) / A;
    lo = fmin(r0, r1);
    hi = fmax(r0, r1);
}

// Padded column interval [x0, x1] of padded row y that can hold accepted
// points of the ray at unpadded pixel (u, v); false if none.  With a
// non-tight footprint this is the whole window row.
HP_HD bool footprint_row(const Footprint& F, const CamFrame& C, int pad, int width, int height, int u, int v,
                         int y, int& x0, int& x1) {
    x0 = u;
    x1 = u + 2 * pad;
    if (!F.tight) return true;
    const double vr = double(y - pad);  // unpadded row index
    const double mb = 1e-3 * C.ph;
    double bb1 = (0.5 * double(height) - vr - 1.0) * C.ph - mb;
    double bb2 = (0.5 * double(height) - vr) * C.ph + mb;
    bb1 = fmax(bb1, F.bmin);
    bb2 = fmin(bb2, F.bmax);
    if (bb1 > bb2) return false;
    double l1, h1, l2, h2;
    footprint_a_at(F, C, bb1, l1, h1);
    footprint_a_at(F, C, bb2, l2, h2);
    const double amin = (F.bL >= bb1 && F.bL <= bb2) ? F.amin : fmin(l1, l2);
    const double amax = (F.bR >= bb1 && F.bR <= bb2) ? F.amax : fmax(h1, h2);
    // columns (padded), clamped to the window before converting to int
    const double lo_win = double(u), hi_win = double(u + 2 * pad);
    const double c0 = floor(amin / C.pw + 0.5 * double(width)) - 1.0 + double(pad);
    const double c1 = floor(amax / C.pw + 0.5 * double(width)) + 1.0 + double(pad);
    if (!(c0 <= hi_win) || !(c1 >= lo_win)) return false;
    x0 = int(fmax(c0, lo_win));
    x1 = int(fmin(c1, hi_win));
    return x0 <= x1;
}

}  // namespace hp
