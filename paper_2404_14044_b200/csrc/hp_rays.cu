// hp_rays.cu — the camera's ray grid generated on the device (SURVEY.md §8f
// row 2): unit directions through the pixel centres, row-major, bit-identical
// to the reference's numpy `ray_grid` (geometry.py:289-306), so the host
// uploads no pixels / directions for a full view.
//
// numpy's evaluation, element by element (separate ufuncs: no contraction):
//   du = ((u + 0.5) - 0.5 W) * pw ;  dv = ((v + 0.5) - 0.5 H) * ph
//   d_k = (f * F_k + du * R_k) - dv * U_k
//   n = sqrt((d_0 * d_0 + d_1 * d_1) + d_2 * d_2)   (add.reduce over 3 items)
//   d_k /= n
// Every operation is IEEE round-to-nearest on the device too (__dmul_rn /
// __dadd_rn / __dsub_rn / __ddiv_rn / sqrt), so the bits agree.
#include "hp_common.cuh"

namespace hp {
namespace {

struct GridCam {
    double f, pw, ph, hw, hh;
    double F[3], R[3], U[3];
    int64_t W;
};

__global__ void k_ray_grid(GridCam c, int64_t m, int64_t v0, double* __restrict__ dirs, int64_t* __restrict__ pixels,
                           double tn, double tf, double* __restrict__ t_near, double* __restrict__ t_far) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < m; k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = v0 * c.W + k;  // grid index (row-major)
        const int64_t u = g % c.W, v = g / c.W;
        const double du = __dmul_rn(__dsub_rn(__dadd_rn(double(u), 0.5), c.hw), c.pw);
        const double dv = __dmul_rn(__dsub_rn(__dadd_rn(double(v), 0.5), c.hh), c.ph);
        double d[3];
#pragma unroll
        for (int x = 0; x < 3; x++)
            d[x] = __dsub_rn(__dadd_rn(__dmul_rn(c.f, c.F[x]), __dmul_rn(du, c.R[x])), __dmul_rn(dv, c.U[x]));
        const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                              __dmul_rn(d[2], d[2])));
#pragma unroll
        for (int x = 0; x < 3; x++) dirs[3 * k + x] = __ddiv_rn(d[x], n);
        if (pixels) {
            pixels[2 * k] = u;
            pixels[2 * k + 1] = v;
        }
        if (t_near) t_near[k] = tn;
        if (t_far) t_far[k] = tf;
    }
}

// glibc's hypot (2.35+, sysdeps/ieee754/dbl-64/e_hypot.c: Borges' corrected
// sqrt, the variant built without FMA), restated operation for operation in
// round-to-nearest so that the device value equals the host libm's bit for
// bit (glibc's hypot is not correctly rounded: a correctly rounded device
// hypot would differ from numpy in ~0.2% of the slopes).  Checked against
// the image's glibc on 2e7 inputs of the slope distribution and of a wide
// range.  Arguments here are finite and far from the
// scaling thresholds (2^-511, 2^511), which are kept for completeness.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ __forceinline__ double glibc_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
        return __ddiv_rn(glibc_hypot_kernel(__dmul_rn(ax, 0x1p-600), __dmul_rn(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay < 0x1p-511) {
        if (ax >= __ddiv_rn(ay, 0x1p-54)) return __dadd_rn(ax, ay);
        return __dmul_rn(glibc_hypot_kernel(__ddiv_rn(ax, 0x1p-600), __ddiv_rn(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay <= __dmul_rn(ax, 0x1p-54)) return __dadd_rn(ax, ay);
    return glibc_hypot_kernel(ax, ay);
}

// geometry.radius_slopes per ray, in numpy's operation order (as
// hp_radius_slopes_host): ox = ((u + 0.5) - W/2) * pw, a2 = ox^2 + oy^2,
// ae2 = f^2 + a2, slope = (f kr) / (sqrt(ae2) * hypot(sqrt(a2) - kr, f)).
__global__ void k_radius_slopes(double f, double pw, double ph, double hw, double hh, int64_t W, int64_t row0,
                                const int64_t* __restrict__ pix, int64_t stride, int64_t m, double kr, int approx,
                                double* __restrict__ out) {
    const double fkr = __dmul_rn(f, kr), ff = __dmul_rn(f, f);
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = row0 * W + r;
        const int64_t pu = pix ? pix[r * stride] : g % W;
        const int64_t pv = pix ? pix[r * stride + 1] : g / W;
        const double ox = __dmul_rn(__dsub_rn(__dadd_rn(double(pu), 0.5), hw), pw);
        const double oy = __dmul_rn(__dsub_rn(__dadd_rn(double(pv), 0.5), hh), ph);
        const double a2 = __dadd_rn(__dmul_rn(ox, ox), __dmul_rn(oy, oy));
        const double ae2 = __dadd_rn(ff, a2);
        out[r] = approx ? __ddiv_rn(fkr, ae2)
                        : __ddiv_rn(fkr, __dmul_rn(__dsqrt_rn(ae2), glibc_hypot(__dsub_rn(__dsqrt_rn(a2), kr), f)));
    }
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_radius_slopes(const hp_camera* cam, int64_t row0, const int64_t* pixels, int64_t pixel_stride,
                                int64_t m, double kernel_radius, int approx, double* slopes, hp_stream_t stream) {
    if (!cam || m < 0 || row0 < 0 || (m > 0 && !slopes) ||
        (!pixels && (cam->width <= 0 || row0 * cam->width + m > cam->width * cam->height))) {
        set_error("hp_radius_slopes: bad arguments");
        return HP_EINVAL;
    }
    if (m == 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    TimedSpan ts("k_radius_slopes", s);
    k_radius_slopes<<<grid_for(m, 256), 256, 0, s>>>(cam->focal_length, cam->pixel_width, cam->pixel_height,
                                                     0.5 * double(cam->width), 0.5 * double(cam->height),
                                                     cam->width, row0, pixels, pixel_stride, m, kernel_radius,
                                                     approx, slopes);
    HP_CHECK_LAUNCH("k_radius_slopes");
    return HP_OK;
}

extern "C" int hp_ray_grid(const hp_camera* cam, int64_t row0, int64_t rows, double* dirs, int64_t* pixels,
                           double t_near_value, double t_far_value, double* t_near, double* t_far,
                           hp_stream_t stream) {
    if (!cam || row0 < 0 || rows < 0 || row0 + rows > cam->height || cam->width < 0) {
        set_error("hp_ray_grid: rows outside the camera");
        return HP_EINVAL;
    }
    const int64_t m = rows * cam->width;
    if (m == 0) return HP_OK;
    if (!dirs) {
        set_error("hp_ray_grid: dirs is NULL");
        return HP_EINVAL;
    }
    GridCam c;
    c.f = cam->focal_length;
    c.pw = cam->pixel_width;
    c.ph = cam->pixel_height;
    c.hw = 0.5 * double(cam->width);
    c.hh = 0.5 * double(cam->height);
    for (int x = 0; x < 3; x++) {
        c.F[x] = cam->forward[x];
        c.R[x] = cam->right[x];
        c.U[x] = cam->up[x];
    }
    c.W = cam->width;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    TimedSpan ts("k_ray_grid", s);
    k_ray_grid<<<grid_for(m, 256), 256, 0, s>>>(c, m, row0, dirs, pixels, t_near_value, t_far_value, t_near, t_far);
    HP_CHECK_LAUNCH("k_ray_grid");
    return HP_OK;
}
