// Host-side check of the query footprint (hp_cone.cuh): for random cameras
// (rotated, off-origin), clouds and rays, every point the reference's fp64
// cone test accepts must sit in a pixel inside the footprint's column
// interval of its row.  Buckets are computed with the build's expressions
// (hp_oracle.c bucket_of order).  Exits 1 on a violation; prints the ratio of
// footprint pixels to window pixels.  Run by tests/test_cone_filter.py.
#include <cstdio>
#include <cstdlib>
#include <random>

#include "../../paper_2404_14044_b200/csrc/hp_cone.cuh"

using namespace hp;

int main(int argc, char** argv) {
    const int scenes = argc > 1 ? atoi(argv[1]) : 40;
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    long bad = 0, accepted = 0;
    double win_px = 0, fp_px = 0;
    for (int sc = 0; sc < scenes; sc++) {
        // camera: random origin near 0, looking at (0,0,4) with random up
        const double ox = (U(rng) - 0.5) * 1.5, oy = (U(rng) - 0.5) * 1.5, oz = (U(rng) - 0.5) * 1.0;
        double fw[3] = {-ox, -oy, 4.0 - oz};
        double n = sqrt(fw[0] * fw[0] + fw[1] * fw[1] + fw[2] * fw[2]);
        for (double& x : fw) x /= n;
        double up0[3] = {U(rng) - 0.5, 1.0, U(rng) - 0.5};
        double rt[3] = {up0[1] * fw[2] - up0[2] * fw[1], up0[2] * fw[0] - up0[0] * fw[2], up0[0] * fw[1] - up0[1] * fw[0]};
        n = sqrt(rt[0] * rt[0] + rt[1] * rt[1] + rt[2] * rt[2]);
        for (double& x : rt) x /= n;
        double up[3] = {fw[1] * rt[2] - fw[2] * rt[1], fw[2] * rt[0] - fw[0] * rt[2], fw[0] * rt[1] - fw[1] * rt[0]};
        const int W = 40 + int(U(rng) * 60), H = 30 + int(U(rng) * 50);
        const double fov = (20.0 + U(rng) * 80.0) * 3.141592653589793 / 180.0;
        const double focal = 0.5 + U(rng);
        const double pw = 2.0 * focal * tan(fov / 2.0) / W;
        const double ph = pw * (0.7 + 0.6 * U(rng));
        const double delta = 0.002 + U(rng) * 0.05;
        // kernel size as the reference derives it (SearchConfig), or random
        const double disc = sqrt(pw * ph / 3.141592653589793);
        const int pad = (sc % 2) ? int(ceil(delta * focal / disc)) : 1 + int(U(rng) * 12);
        CamFrame C;
        for (int k = 0; k < 3; k++) { C.r[k] = rt[k]; C.u[k] = up[k]; C.f[k] = fw[k]; }
        C.focal = focal; C.pw = pw; C.ph = ph; C.half_w = 0.5 * W; C.half_h = 0.5 * H;
        // points: shell + box around (0,0,4)
        const int npts = 20000;
        std::vector<double> P(3 * npts);
        std::vector<int> row(npts), col(npts);
        const int wp = W + 2 * pad, hp = H + 2 * pad;
        for (int i = 0; i < npts; i++) {
            double x = (U(rng) - 0.5) * 3, y = (U(rng) - 0.5) * 3, z = 4 + (U(rng) - 0.5) * 3;
            P[3 * i] = x - ox; P[3 * i + 1] = y - oy; P[3 * i + 2] = z - oz;
            const double p0 = P[3 * i], p1 = P[3 * i + 1], p2 = P[3 * i + 2];
            const double depth = (p0 * fw[0] + p1 * fw[1]) + p2 * fw[2];
            const double a = (p0 * rt[0] + p1 * rt[1]) + p2 * rt[2];
            const double b = (p0 * up[0] + p1 * up[1]) + p2 * up[2];
            const double s = focal / depth;
            const double uu = (a * s) / pw + 0.5 * W, vv = ((-b) * s) / ph + 0.5 * H;
            const double fu = floor(uu) + pad, fv = floor(vv) + pad;
            const bool ok = depth > 0 && fu >= 0 && fu < wp && fv >= 0 && fv < hp;
            row[i] = ok ? int(fv) : -1;
            col[i] = ok ? int(fu) : -1;
        }
        for (int ray = 0; ray < 200; ray++) {
            const int u = int(U(rng) * W), v = int(U(rng) * H);
            const double du = (u + 0.5 - 0.5 * W) * pw, dv = (v + 0.5 - 0.5 * H) * ph;
            double d[3];
            for (int k = 0; k < 3; k++) d[k] = focal * fw[k] + du * rt[k] - dv * up[k];
            n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            for (double& x : d) x /= n;
            const double kr = delta * focal / 1.0;
            const double a2 = du * du + dv * dv, ae2 = focal * focal + a2;
            const double slope = focal * kr / (sqrt(ae2) * hypot(sqrt(a2) - kr, focal));
            RayParams r{};
            r.d0 = d[0]; r.d1 = d[1]; r.d2 = d[2]; r.tn = 0.5; r.tf = 20.0; r.slope = slope;
            Footprint Fp;
            footprint_init(Fp, C, d[0], d[1], d[2], slope);
            for (int y = v; y < v + 2 * pad + 1; y++) {
                int x0, x1;
                if (footprint_row(Fp, C, pad, W, H, u, v, y, x0, x1)) fp_px += x1 - x0 + 1;
                win_px += 2 * pad + 1;
            }
            // adversarial points right at the cone surface of this ray
            const double th0 = atan(slope);
            double e1[3] = {-d[1], d[0], 0.0};
            double en = sqrt(e1[0] * e1[0] + e1[1] * e1[1]);
            for (double& x : e1) x /= en;
            double e2[3] = {d[1] * e1[2] - d[2] * e1[1], d[2] * e1[0] - d[0] * e1[2], d[0] * e1[1] - d[1] * e1[0]};
            for (int a = 0; a < 400; a++) {
                const double th = th0 * (1.0 + (U(rng) - 0.5) * 2e-6), ph_ = U(rng) * 6.283185307179586;
                const double tt = 0.6 + U(rng) * 15.0;
                double q[3];
                for (int k = 0; k < 3; k++)
                    q[k] = tt * (cos(th) * d[k] + sin(th) * (cos(ph_) * e1[k] + sin(ph_) * e2[k]));
                const double depth = (q[0] * fw[0] + q[1] * fw[1]) + q[2] * fw[2];
                const double aa = (q[0] * rt[0] + q[1] * rt[1]) + q[2] * rt[2];
                const double bb = (q[0] * up[0] + q[1] * up[1]) + q[2] * up[2];
                const double ss = focal / depth;
                const double fu = floor((aa * ss) / pw + 0.5 * W) + pad, fv = floor(((-bb) * ss) / ph + 0.5 * H) + pad;
                if (!(depth > 0 && fu >= 0 && fu < wp && fv >= 0 && fv < hp)) continue;
                const int rr = int(fv), cc = int(fu);
                if (rr < v || rr > v + 2 * pad || cc < u || cc > u + 2 * pad) continue;
                double t2, dd2;
                if (!cone_test(q[0], q[1], q[2], r, t2, dd2)) continue;
                accepted++;
                int x0, x1;
                const bool any = footprint_row(Fp, C, pad, W, H, u, v, rr, x0, x1);
                if (!any || cc < x0 || cc > x1) {
                    if (bad < 5) printf("violation (surface): ray (%d,%d) row %d col %d range [%d,%d]\n", u, v, rr, cc, x0, x1);
                    bad++;
                }
            }
            for (int i = 0; i < npts; i++) {
                if (row[i] < v || row[i] > v + 2 * pad || col[i] < u || col[i] > u + 2 * pad) continue;
                double t, d2;
                if (!cone_test(P[3 * i], P[3 * i + 1], P[3 * i + 2], r, t, d2)) continue;
                accepted++;
                int x0, x1;
                const bool any = footprint_row(Fp, C, pad, W, H, u, v, row[i], x0, x1);
                if (!any || col[i] < x0 || col[i] > x1) {
                    if (bad < 5)
                        printf("violation: scene %d ray (%d,%d) row %d col %d range [%d,%d] any=%d tight=%d\n", sc, u, v,
                               row[i], col[i], x0, x1, int(any), Fp.tight);
                    bad++;
                }
            }
        }
    }
    printf("accepted=%ld violations=%ld footprint/window=%.3f\n", accepted, bad, fp_px / win_px);
    return bad ? 1 : 0;
}
