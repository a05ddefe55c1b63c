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
HP_HD bool cone_test(double p0, double p1, double p2, const RayParams& r,
                                          double& t, double& dist2) {
    t = cadd(cadd(cmul(p0, r.d0), cmul(p1, r.d1)), cmul(p2, r.d2));
    if (t < r.tn || t > r.tf) return false;
    const double e0 = csub(p0, cmul(t, r.d0));
    const double e1 = csub(p1, cmul(t, r.d1));
    const double e2 = csub(p2, cmul(t, r.d2));
    dist2 = cadd(cadd(cmul(e0, e0), cmul(e1, e1)), cmul(e2, e2));
    const double rad = cmul(t, r.slope);
    return !(dist2 > cmul(rad, rad));
}

// float32 filter.  P = (x, y, z, e) with e = 2^-18 |p|_1 (rounded up).  The
// band eps = e * max(1, slope) + 2^-22 * t_far bounds |t32 - t64| and the
// error of the fp32 perpendicular distance (derivation in DESIGN.md).
// Returns 0 = reject, 1 = accept, 2 = decide in fp64.
HP_HD int cone_filter(const float4 P, const RayParams& r) {
    const float eps = fmaf(P.w, r.smax, r.eps_ray);
    const float t = fmaf(P.z, r.f2, fmaf(P.y, r.f1, P.x * r.f0));
    if (t < r.ftn - eps || t > r.ftf + eps) return 0;
    const float ex = fmaf(-t, r.f0, P.x), ey = fmaf(-t, r.f1, P.y), ez = fmaf(-t, r.f2, P.z);
    const float d2 = fmaf(ez, ez, fmaf(ey, ey, ex * ex));
    const float rr = t * r.fslope;
    const float hi = rr + eps;
    if (d2 > hi * hi * (1.0f + 0x1p-20f)) return 0;
    const float lo = rr - eps;
    const bool t_in = (t >= r.ftn + eps) && (t <= r.ftf - eps);
    if (t_in && lo > 0.0f && d2 < lo * lo * (1.0f - 0x1p-20f)) return 1;
    return 2;
}


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

}  // namespace hp
