// Host-side soundness stress of the float32 cone filter (hp_cone.cuh): for
// millions of (ray, point) pairs placed adversarially close to the cone and
// t-range boundaries, a "sure accept" must be accepted by the reference fp64
// test and a "sure reject" must be rejected by it.  Prints the counts; exits
// 1 on any violation.  Built and run by tests/test_cone_filter.py (CPU).
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../../paper_2404_14044_b200/csrc/hp_cone.cuh"

using namespace hp;

int main(int argc, char** argv) {
    const long n = argc > 1 ? atol(argv[1]) : 2000000;
    std::mt19937_64 rng(12345);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    long sure_acc = 0, sure_rej = 0, unsure = 0, bad = 0, acc = 0;
    for (long k = 0; k < n; k++) {
        // ray: random direction within ~35 degrees of +z, random t range and slope
        double dx = (U(rng) - 0.5) * 1.4, dy = (U(rng) - 0.5) * 1.4, dz = 1.0;
        const double nrm = sqrt(dx * dx + dy * dy + dz * dz);
        RayParams r{};
        r.d0 = dx / nrm;
        r.d1 = dy / nrm;
        r.d2 = dz / nrm;
        r.tn = 0.1 + U(rng) * 2.0;
        r.tf = r.tn + 0.5 + U(rng) * 20.0;
        const int sk = int(U(rng) * 4);
        r.slope = sk == 0 ? U(rng) * 1e-3 : sk == 1 ? U(rng) * 0.05 : sk == 2 ? U(rng) * 0.5 : U(rng) * 3.0;
        ray_derive(r);
        // point: t near a boundary or inside, perpendicular offset near r(t)
        const int mode = int(U(rng) * 5);
        double t;
        if (mode == 0) t = r.tn + (U(rng) - 0.5) * 1e-5 * r.tn;
        else if (mode == 1) t = r.tf + (U(rng) - 0.5) * 1e-5 * r.tf;
        else t = r.tn + U(rng) * (r.tf - r.tn);
        const double rad = t * r.slope;
        double off;
        const int om = int(U(rng) * 4);
        if (om == 0) off = rad * (1.0 + (U(rng) - 0.5) * 1e-5);
        else if (om == 1) off = rad * (1.0 + (U(rng) - 0.5) * 1e-3);
        else off = rad * U(rng) * 1.5;
        // unit vector orthogonal to d
        double ax = -r.d1, ay = r.d0, az = 0.0;
        double an = sqrt(ax * ax + ay * ay);
        if (an < 1e-12) { ax = 1; ay = 0; an = 1; }
        ax /= an; ay /= an;
        const double bx = r.d1 * az - r.d2 * ay, by = r.d2 * ax - r.d0 * az, bz = r.d0 * ay - r.d1 * ax;
        const double ph = U(rng) * 6.283185307179586;
        const double ox = off * (cos(ph) * ax + sin(ph) * bx), oy = off * (cos(ph) * ay + sin(ph) * by),
                     oz = off * (cos(ph) * az + sin(ph) * bz);
        // world offset of the camera origin (points are origin-relative)
        const double p0 = t * r.d0 + ox, p1 = t * r.d1 + oy, p2 = t * r.d2 + oz;
        double tt, d2;
        const bool ref = cone_test(p0, p1, p2, r, tt, d2);
        const float4 P = filter_point(p0, p1, p2);
        const int cls = cone_filter(P, r);
        acc += ref;
        if (cls == 1) { sure_acc++; if (!ref) bad++; }
        else if (cls == 0) { sure_rej++; if (ref) bad++; }
        else unsure++;
        if (bad == 1 && (cls == 1) != ref && cls != 2) {
            printf("violation: cls=%d ref=%d t=%.17g tn=%.17g tf=%.17g slope=%.17g\n", cls, int(ref), tt, r.tn, r.tf, r.slope);
            bad++;
        }
    }
    printf("pairs=%ld accepted=%ld sure_accept=%ld sure_reject=%ld uncertain=%ld violations=%ld\n", n, acc, sure_acc,
           sure_rej, unsure, bad);
    return bad ? 1 : 0;
}
