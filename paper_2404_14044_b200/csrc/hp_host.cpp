// hp_host.cpp — host-side helpers of the path that stay on the CPU by design.
//
// hp_radius_slopes_host: the reference's vectorised radius_slopes
// (geometry.py:249-260) with the same operation order and
// the same libm calls numpy makes (sqrt; hypot from glibc), so the values are
// bit-identical to `radius_slopes` in numpy; compiled without FP contraction.
// Kept on the host on purpose: hypot is not correctly rounded, so a device
// version could differ in the last bit.  Runs on host threads.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "../../include/hashpoint_b200.h"

namespace {

void slopes_range(const hp_camera& c, const int64_t* pix, int64_t stride, double kr, int approx, double* out,
                  int64_t a, int64_t b) {
    const double f = c.focal_length;
    const double hw = 0.5 * double(c.width), hh = 0.5 * double(c.height);
    const double fkr = f * kr;
    const double ff = f * f;
    for (int64_t r = a; r < b; r++) {
        // pixels NULL: the ray grid, ray r = pixel (r % W, r / W)
        const int64_t pu = pix ? pix[r * stride] : r % c.width;
        const int64_t pv = pix ? pix[r * stride + 1] : r / c.width;
        // _plane_offsets: (u + 0.5 - 0.5 * W) * pixel_width (left to right)
        const double ox = ((double(pu) + 0.5) - hw) * c.pixel_width;
        const double oy = ((double(pv) + 0.5) - hh) * c.pixel_height;
        const double a2 = ox * ox + oy * oy;
        const double ae2 = ff + a2;
        out[r] = approx ? fkr / ae2 : fkr / (std::sqrt(ae2) * std::hypot(std::sqrt(a2) - kr, f));
    }
}

}  // namespace

extern "C" int hp_radius_slopes_host(const hp_camera* cam, const int64_t* pixels, int64_t pixel_stride, int64_t m,
                                     double kernel_radius, int approx, double* slopes, int threads) {
    if (!cam || m < 0 || (m > 0 && !slopes) || (!pixels && m > cam->width * cam->height)) return HP_EINVAL;
    if (threads < 1) threads = 1;
    const int64_t per = (m + threads - 1) / threads;
    if (threads == 1 || m < 4096) {
        slopes_range(*cam, pixels, pixel_stride, kernel_radius, approx, slopes, 0, m);
        return HP_OK;
    }
    std::vector<std::thread> pool;
    for (int k = 0; k < threads; k++) {
        const int64_t a = k * per, b = std::min<int64_t>(m, a + per);
        if (a >= b) break;
        pool.emplace_back(slopes_range, std::cref(*cam), pixels, pixel_stride, kernel_radius, approx, slopes, a, b);
    }
    for (auto& t : pool) t.join();
    return HP_OK;
}

// hp_host_upload: pageable host memory -> device through a pinned staging
// buffer.  Host threads claim pieces in order and copy them into the staging
// buffer; the calling thread enqueues each piece's DMA as soon as it is
// staged, so the host copies, the DMA and the caller's stream overlap (the
// driver's own pageable path stages through a few small buffers on one
// thread: ~11-20 GB/s on the B200 box).
extern "C" int hp_host_upload(void* dst, const void* src, size_t bytes, void* staging, size_t piece, int threads,
                              cudaStream_t stream) {
    if (bytes == 0) return HP_OK;
    if (!dst || !src || !staging) return HP_EINVAL;
    if (piece == 0) piece = size_t(2) << 20;
    if (threads < 1) threads = 1;
    const size_t n = (bytes + piece - 1) / piece;
    auto* dsrc = static_cast<const char*>(src);
    auto* dstg = static_cast<char*>(staging);
    std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[n]);
    for (size_t k = 0; k < n; k++) done[k].store(0, std::memory_order_relaxed);
    std::atomic<size_t> next{0};
    auto work = [&]() {
        for (size_t k; (k = next.fetch_add(1, std::memory_order_relaxed)) < n;) {
            const size_t off = k * piece, len = std::min(piece, bytes - off);
            std::memcpy(dstg + off, dsrc + off, len);
            done[k].store(1, std::memory_order_release);
        }
    };
    std::vector<std::thread> pool;
    const int nt = int(std::min<size_t>(size_t(threads), n));
    for (int t = 0; t < nt; t++) pool.emplace_back(work);
    int rc = HP_OK;
    for (size_t k = 0; k < n; k++) {
        while (!done[k].load(std::memory_order_acquire)) std::this_thread::yield();
        const size_t off = k * piece, len = std::min(piece, bytes - off);
        if (rc == HP_OK &&
            cudaMemcpyAsync(static_cast<char*>(dst) + off, dstg + off, len, cudaMemcpyHostToDevice, stream) !=
                cudaSuccess)
            rc = HP_ECUDA;
    }
    for (auto& t : pool) t.join();
    return rc;
}
