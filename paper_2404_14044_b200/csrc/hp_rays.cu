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

}  // namespace
}  // namespace hp

using namespace hp;

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
