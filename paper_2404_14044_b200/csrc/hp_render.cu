// hp_render.cu — colour and depth synthesis from the retained samples
// (reference renderer.py:72-192), one thread per ray.
//
//   volume: each retained sample gets a density over its segment (deltas from
//     consecutive t, the last one repeated, t_far - t for a single sample),
//     sigma = -log1p(-alpha) / delta, passed = exp(-sigma delta), weight =
//     T * (1 - passed) (alpha >= 1: opaque; delta <= 0: alpha itself);
//     colour = sum w * sample colour + T * background, depth = sum w t / sum w
//     (t_far when sum w = 0 or the ray retained nothing).
//   knp: the k smallest perpendicular distances (ties: sample order), weights
//     1/d or the on-ray points alone, normalised; colour = sum w * point
//     colour, depth = sum w t; rays that retained nothing leave the pixel.
//
// Several rays on one pixel: the last ray wins, as in the reference's loop
// (k_render_owner records the largest ray index per pixel first).
// Values go through log1p / exp / divisions whose last bits may differ from
// glibc / numpy; compare at rtol 1e-12.
#include <cmath>

#include "hp_common.cuh"

namespace hp {
namespace {

struct RenderArgs {
    const int64_t* r_off;
    const int64_t* r_id;
    const double* r_t;
    const double* r_dist;
    const double* r_alpha;
    const double* r_color;       // [R, 3] (volume)
    const double* point_colors;  // [n, 3] (knp)
    const int64_t* pixels;
    int64_t stride;
    const double* t_far;
    int64_t m, width;
    int knp, knp_k;
    double bg[3];
    const int* owner;
    double* color;  // [H, W, 3]
    double* depth;  // [H, W]
};

__global__ void k_render_owner(const int64_t* __restrict__ pixels, int64_t stride, int64_t m, int64_t width,
                               int* __restrict__ owner) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < m; r += int64_t(gridDim.x) * blockDim.x)
        atomicMax(owner + pixels[r * stride + 1] * width + pixels[r * stride], int(r));
}

__global__ void k_render(RenderArgs A) {
    for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < A.m; r += int64_t(gridDim.x) * blockDim.x) {
        const int64_t pix = A.pixels[r * A.stride + 1] * A.width + A.pixels[r * A.stride];
        if (A.owner[pix] != int(r)) continue;  // a later ray owns this pixel
        const int64_t lo = A.r_off[r], hi = A.r_off[r + 1];
        const int n = int(hi - lo);
        const double tf = A.t_far[r];
        double* out = A.color + 3 * pix;
        if (!A.knp) {
            if (n == 0) {
                for (int c = 0; c < 3; c++) out[c] = A.bg[c];
                A.depth[pix] = tf;
                continue;
            }
            double trans = 1.0, acc[3] = {0.0, 0.0, 0.0}, wt = 0.0, ws = 0.0;
            for (int j = 0; j < n; j++) {
                const double a = A.r_alpha[lo + j], tj = A.r_t[lo + j];
                double dt;
                if (n == 1)
                    dt = __dsub_rn(tf, tj);
                else if (j + 1 < n)
                    dt = __dsub_rn(A.r_t[lo + j + 1], tj);
                else
                    dt = __dsub_rn(tj, A.r_t[lo + j - 1]);
                double absorbed, passed;
                if (a >= 1.0) {
                    absorbed = 1.0;
                    passed = 0.0;
                } else if (dt > 0.0) {
                    const double sigma = __ddiv_rn(-log1p(-a), dt);
                    passed = exp(-__dmul_rn(sigma, dt));
                    absorbed = __dsub_rn(1.0, passed);
                } else {
                    absorbed = a;
                    passed = __dsub_rn(1.0, a);
                }
                const double w = __dmul_rn(trans, absorbed);
                trans = __dmul_rn(trans, passed);
                for (int c = 0; c < 3; c++) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, A.r_color[3 * (lo + j) + c]));
                wt = __dadd_rn(wt, __dmul_rn(w, tj));
                ws = __dadd_rn(ws, w);
            }
            for (int c = 0; c < 3; c++) out[c] = __dadd_rn(acc[c], __dmul_rn(trans, A.bg[c]));
            A.depth[pix] = ws > 0.0 ? __ddiv_rn(wt, ws) : tf;
            continue;
        }
        if (n == 0) continue;  // knp: the pixel keeps the blank image
        const int k = A.knp_k < n ? A.knp_k : n;
        // pass 1: the k-th smallest (d, j) and whether a selected point is on the ray
        double pd = -1.0;
        int pj = -1;
        bool zero = false;
        double wsum = 0.0;
        for (int s = 0; s < k; s++) {  // next smallest (d, j) after (pd, pj)
            double bd = INFINITY;
            int bj = -1;
            for (int j = 0; j < n; j++) {
                const double d = A.r_dist[lo + j];
                const bool after = d > pd || (d == pd && j > pj);
                if (after && (bj < 0 || d < bd || (d == bd && j < bj))) {
                    bd = d;
                    bj = j;
                }
            }
            pd = bd;
            pj = bj;
            zero |= bd == 0.0;
        }
        const double dk = pd;
        const int jk = pj;
        auto selected = [&](double d, int j) { return d < dk || (d == dk && j <= jk); };
        for (int j = 0; j < n; j++) {
            const double d = A.r_dist[lo + j];
            if (selected(d, j)) wsum = __dadd_rn(wsum, zero ? (d == 0.0 ? 1.0 : 0.0) : __ddiv_rn(1.0, d));
        }
        double acc[3] = {0.0, 0.0, 0.0}, dep = 0.0;
        for (int j = 0; j < n; j++) {
            const double d = A.r_dist[lo + j];
            if (!selected(d, j)) continue;
            const double w = __ddiv_rn(zero ? (d == 0.0 ? 1.0 : 0.0) : __ddiv_rn(1.0, d), wsum);
            const int64_t id = A.r_id[lo + j];
            for (int c = 0; c < 3; c++) acc[c] = __dadd_rn(acc[c], __dmul_rn(w, A.point_colors[3 * id + c]));
            dep = __dadd_rn(dep, __dmul_rn(w, A.r_t[lo + j]));
        }
        for (int c = 0; c < 3; c++) out[c] = acc[c];
        A.depth[pix] = dep;
    }
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_render(int mode, const int64_t* r_off, int64_t m, const int64_t* r_id, const double* r_t,
                         const double* r_dist, const double* r_alpha, const double* r_color,
                         const double* point_colors, const int64_t* pixels, int64_t pixel_stride,
                         const double* t_far, int32_t knp_k, const double* background, int64_t width,
                         int64_t height, int32_t* owner, double* color, double* depth, hp_stream_t stream) {
    if ((mode != 0 && mode != 1) || m < 0 || width < 0 || height < 0 || !background || (mode == 1 && knp_k < 1)) {
        set_error("hp_render: invalid arguments");
        return HP_EINVAL;
    }
    if (m == 0) return HP_OK;
    if (!r_off || !pixels || !t_far || !owner || !color || !depth || m >= (int64_t(1) << 31)) {
        set_error("hp_render: invalid arguments");
        return HP_EINVAL;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(owner, 0xff, size_t(width * height) * sizeof(int32_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_render memset");
    RenderArgs A{r_off, r_id, r_t, r_dist, r_alpha, r_color, point_colors, pixels, pixel_stride, t_far, m, width,
                 mode, knp_k, {background[0], background[1], background[2]}, owner, color, depth};
    TimedSpan ts("k_render", s);
    k_render_owner<<<grid_for(m, 256), 256, 0, s>>>(pixels, pixel_stride, m, width, owner);
    HP_CHECK_LAUNCH("k_render_owner");
    k_render<<<grid_for(m, 128), 128, 0, s>>>(A);
    HP_CHECK_LAUNCH("k_render");
    return HP_OK;
}
