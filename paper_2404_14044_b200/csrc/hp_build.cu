// hp_build.cu — hash-index build: project -> warp-aggregated histogram ->
// Morton-order exclusive scan -> counting-sort scatter -> per-bucket id order
// -> slot gather (+ row-major query layout).
//
// Reference: hash_index.build (hash_index.py:151-190), rasterize_points
// (:95-112), morton_codes (:81-92), _kernels.scatter_by_bucket
// (_kernels.py:76-83).  Output arrays are bit-identical to the reference's:
// buckets are computed with the same fp64 expressions (fixed order, no FMA;
// see DESIGN.md "projection"), table starts follow the Morton order of the
// padded pixel grid, empty pixels get start 0, and points inside a pixel are
// ordered by ascending original index.
#include <climits>

#include "hp_common.cuh"
#include "hp_cone.cuh"
#include "hp_sortnet.cuh"

namespace hp {
namespace {

struct CamDev {
    double o[3], r[3], u[3], f[3];
    double focal, pw, ph, half_w, half_h;
};

constexpr int kProjThreads = 256;

constexpr int kSmallBucket = 32;

// Bucket (row-major padded pixel) of one point; -1 if not rasterized.
// Same expressions and evaluation order as the oracle (hp_oracle.c bucket_of)
// and the reference's Camera.project + rasterize_points.
__device__ __forceinline__ int32_t bucket_of(const CamDev& c, double x, double y, double z,
                                             int pad, int wp, int hp) {
    const double p0 = dsub(x, c.o[0]), p1 = dsub(y, c.o[1]), p2 = dsub(z, c.o[2]);
    const double depth = dadd(dadd(dmul(p0, c.f[0]), dmul(p1, c.f[1])), dmul(p2, c.f[2]));
    const double a = dadd(dadd(dmul(p0, c.r[0]), dmul(p1, c.r[1])), dmul(p2, c.r[2]));
    const double b = dadd(dadd(dmul(p0, c.u[0]), dmul(p1, c.u[1])), dmul(p2, c.u[2]));
    const double s = __ddiv_rn(c.focal, depth);
    const double u = dadd(__ddiv_rn(dmul(a, s), c.pw), c.half_w);
    const double v = dadd(__ddiv_rn(dmul(-b, s), c.ph), c.half_h);
    const double fu = dadd(floor(u), double(pad));
    const double fv = dadd(floor(v), double(pad));
    const bool ok = depth > 0.0 && fu >= 0.0 && fu < double(wp) && fv >= 0.0 && fv < double(hp);
    return ok ? int32_t(fv) * wp + int32_t(fu) : -1;
}

// Pass 1+2: project every point (xyz staged through shared memory with
// 16-byte vector loads) and build the per-pixel histogram with warp-aggregated
// atomics (lanes hitting the same pixel elect one leader).
__global__ void __launch_bounds__(kProjThreads) k_project(const double* __restrict__ xyz, int64_t n,
                                                          CamDev cam, int pad, int wp, int hp,
                                                          int32_t* __restrict__ lin,
                                                          int32_t* __restrict__ cnt, int row0 = 0,
                                                          int row1 = INT_MAX) {
    __shared__ __align__(16) double tile[kProjThreads * 3];
    for (int64_t base = int64_t(blockIdx.x) * kProjThreads; base < n;
         base += int64_t(gridDim.x) * kProjThreads) {
        const int64_t pts = n - base < kProjThreads ? n - base : kProjThreads;
        const double* src = xyz + base * 3;
        const int64_t words = pts * 3;
        if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
            const double2* s2 = reinterpret_cast<const double2*>(src);
            double2* t2 = reinterpret_cast<double2*>(tile);
            for (int64_t k = threadIdx.x; k < words / 2; k += kProjThreads) t2[k] = __ldg(s2 + k);
            if ((words & 1) && threadIdx.x == 0) tile[words - 1] = src[words - 1];
        } else {
            for (int64_t k = threadIdx.x; k < words; k += kProjThreads) tile[k] = src[k];
        }
        __syncthreads();
        const int64_t i = base + threadIdx.x;
        int32_t l = -1;
        if (threadIdx.x < pts) {
            l = bucket_of(cam, tile[3 * threadIdx.x], tile[3 * threadIdx.x + 1],
                          tile[3 * threadIdx.x + 2], pad, wp, hp);
            if (l >= 0 && (l / wp < row0 || l / wp >= row1)) l = -1;  // outside the row window
            lin[i] = l;
        }
        const unsigned act = __ballot_sync(0xffffffffu, l >= 0);
        if (l >= 0) {
            const unsigned peers = __match_any_sync(act, l);
            if (lane_id() == __ffs(peers) - 1) atomicAdd(&cnt[l], __popc(peers));
        }
        __syncthreads();
    }
}

// Rank of padded pixel (u, v) in the Morton order of the wp x hp grid: the
// number of in-grid pixels with a smaller interleaved code (u bits even, v
// bits odd).  Walks the quadtree from the top level and adds the in-grid area
// of the quadrants that precede the pixel's quadrant at every level.
__device__ __forceinline__ int64_t morton_rank(int u, int v, int wp, int hp, int levels) {
    int64_t rank = 0;
    int bu = 0, bv = 0;
    for (int lv = levels - 1; lv >= 0; --lv) {
        const int h = 1 << lv;
        const int q = ((u >> lv) & 1) | (((v >> lv) & 1) << 1);
        for (int k = 0; k < q; k++) {
            const int x0 = bu + (k & 1) * h, y0 = bv + (k >> 1) * h;
            const int64_t w = x0 < wp ? (x0 + h < wp ? h : wp - x0) : 0;
            const int64_t hh = y0 < hp ? (y0 + h < hp ? h : hp - y0) : 0;
            rank += w * hh;
        }
        bu += (q & 1) * h;
        bv += (q >> 1) * h;
    }
    return rank;
}

__global__ void k_morton_permute(int wp, int hp, int levels, const int32_t* __restrict__ cnt,
                                 int32_t* __restrict__ mrank, int32_t* __restrict__ mcnt) {
    const int64_t P = int64_t(wp) * hp;
    for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < P;
         l += int64_t(gridDim.x) * blockDim.x) {
        const int u = int(l % wp), v = int(l / wp);
        const int32_t r = int32_t(morton_rank(u, v, wp, hp, levels));
        mrank[l] = r;
        mcnt[r] = cnt[l];
    }
}

// Reference tables (int64) + scatter cursors + N_in.
__global__ void k_tables(int64_t P, const int32_t* __restrict__ cnt, const int32_t* __restrict__ mrank,
                         const int32_t* __restrict__ mstart, int64_t* __restrict__ table_start,
                         int64_t* __restrict__ table_count, int32_t* __restrict__ cursor,
                         const int32_t* __restrict__ row_ptr, int64_t* __restrict__ n_in) {
    for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < P;
         l += int64_t(gridDim.x) * blockDim.x) {
        const int32_t c = cnt[l], s = mstart[mrank[l]];
        table_count[l] = c;
        table_start[l] = c ? s : 0;
        cursor[l] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_in = row_ptr[P];
}

// Pass 3: counting-sort scatter (warp-aggregated cursor bumps).  The order
// inside a bucket is fixed afterwards by k_bucket_order.
__global__ void k_scatter(int64_t n, const int32_t* __restrict__ lin, int32_t* __restrict__ cursor,
                          int32_t* __restrict__ slot_pid) {
    for (int64_t base = blockIdx.x * int64_t(blockDim.x); base < n;
         base += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const int32_t l = i < n ? lin[i] : -1;
        const unsigned act = __ballot_sync(0xffffffffu, l >= 0);
        if (l >= 0) {
            const unsigned peers = __match_any_sync(act, l);
            const int leader = __ffs(peers) - 1;
            int32_t pos = 0;
            if (lane_id() == leader) pos = atomicAdd(&cursor[l], __popc(peers));
            pos = __shfl_sync(peers, pos, leader);
            pos += __popc(peers & ((1u << lane_id()) - 1));
            HP_ASSERT(pos >= 0 && pos < n);
            slot_pid[pos] = int32_t(i);
        }
    }
}

// Ascending original id inside every bucket (the reference's scatter is
// stable in input order, _kernels.py:76-83).  Small buckets: insertion sort
// by one thread; large ones are queued for k_big_bucket_order.
__global__ void k_bucket_order(int64_t P, const int64_t* __restrict__ table_start,
                               const int64_t* __restrict__ table_count, int32_t* __restrict__ slot_pid,
                               int32_t* __restrict__ big_list, int32_t* __restrict__ big_n) {
    for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < P;
         l += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = table_count[l];
        if (c < 2) continue;
        if (c > kSmallBucket) {
            big_list[atomicAdd(big_n, 1)] = int32_t(l);
            continue;
        }
        int32_t* seg = slot_pid + table_start[l];
        for (int64_t k = 1; k < c; k++) {  // insertion sort, L1-resident segment
            const int32_t x = seg[k];
            int64_t b = k - 1;
            while (b >= 0 && seg[b] > x) {
                seg[b + 1] = seg[b];
                b--;
            }
            seg[b + 1] = x;
        }
    }
}

__global__ void __launch_bounds__(512) k_big_bucket_order(const int64_t* __restrict__ table_start,
                                                           const int64_t* __restrict__ table_count,
                                                           int32_t* __restrict__ slot_pid,
                                                           const int32_t* __restrict__ big_list,
                                                           const int32_t* __restrict__ big_n) {
    for (int b = blockIdx.x; b < *big_n; b += gridDim.x) {
        const int32_t l = big_list[b];
        int32_t* seg = slot_pid + table_start[l];
        const int64_t c = table_count[l];
        block_bitonic_sort(
            c, [&](int64_t x, int64_t y) { return seg[x] < seg[y]; },
            [&](int64_t x, int64_t y) { int32_t t = seg[x]; seg[x] = seg[y]; seg[y] = t; });
        __syncthreads();
    }
}

// One 32-byte record per slot: (x, y, z) origin-relative and the id (int64 bits).
__device__ __forceinline__ void store_rel4(double* rel4, int64_t k, double x, double y, double z, int32_t id) {
    double4* p = reinterpret_cast<double4*>(rel4) + k;
    *p = make_double4(x, y, z, __longlong_as_double((long long)id));
}

// Slot gather (reference HashIndex slot_x/y/z, reordered_ids) and the
// row-major query layout (origin-relative coordinates).
__global__ void k_gather(int64_t n_cap, const int64_t* __restrict__ n_in_dev, const double* __restrict__ xyz,
                         const int32_t* __restrict__ slot_pid, const int32_t* __restrict__ lin,
                         const int64_t* __restrict__ table_start, double o0, double o1, double o2,
                         int64_t* __restrict__ reordered_ids, double* __restrict__ slot_x,
                         double* __restrict__ slot_y, double* __restrict__ slot_z,
                         hp_query_layout L) {
    const int64_t n_in = *n_in_dev;
    for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < n_in && s < n_cap;
         s += int64_t(gridDim.x) * blockDim.x) {
        const int32_t id = slot_pid[s];
        const double x = xyz[3 * int64_t(id)], y = xyz[3 * int64_t(id) + 1], z = xyz[3 * int64_t(id) + 2];
        reordered_ids[s] = id;
        slot_x[s] = x;
        slot_y[s] = y;
        slot_z[s] = z;
        const int32_t l = lin[id];
        const int64_t rm = int64_t(L.row_ptr[l]) + (s - table_start[l]);
        const double rx = dsub(x, o0), ry = dsub(y, o1), rz = dsub(z, o2);
        L.rel_x[rm] = rx;
        L.rel_y[rm] = ry;
        L.rel_z[rm] = rz;
        L.point_id[rm] = id;
        reinterpret_cast<float4*>(L.relf)[rm] = filter_point(rx, ry, rz);
        store_rel4(L.rel4, rm, rx, ry, rz, id);
    }
}

// Re-layout of an existing HashIndex (reference arrays) into the query layout.
__global__ void k_layout_counts(int64_t P, const int64_t* __restrict__ table_count, int32_t* __restrict__ cnt) {
    for (int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; l < P;
         l += int64_t(gridDim.x) * blockDim.x)
        cnt[l] = int32_t(table_count[l]);
}

__global__ void k_layout_fill(int64_t P, const int64_t* __restrict__ table_start,
                              const int64_t* __restrict__ table_count, const double* __restrict__ sx,
                              const double* __restrict__ sy, const double* __restrict__ sz,
                              const int64_t* __restrict__ sid, double o0, double o1, double o2,
                              hp_query_layout L) {
    // one warp per pixel
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t l = blockIdx.x * int64_t(blockDim.x >> 5) + warp_id(); l < P; l += warps) {
        const int64_t c = table_count[l];
        if (c == 0) continue;
        const int64_t s0 = table_start[l], r0 = L.row_ptr[l];
        for (int64_t k = lane_id(); k < c; k += 32) {
            const double rx = dsub(sx[s0 + k], o0), ry = dsub(sy[s0 + k], o1), rz = dsub(sz[s0 + k], o2);
            L.rel_x[r0 + k] = rx;
            L.rel_y[r0 + k] = ry;
            L.rel_z[r0 + k] = rz;
            L.point_id[r0 + k] = int32_t(sid[s0 + k]);
            reinterpret_cast<float4*>(L.relf)[r0 + k] = filter_point(rx, ry, rz);
            store_rel4(L.rel4, r0 + k, rx, ry, rz, int32_t(sid[s0 + k]));
        }
    }
}

// ---------------------------------------------------------------- scatter_by_bucket
// The reference operator on its own (_kernels.py:76-83): out_ids[cursor[b]++]
// = orig_ids[j] for j in input order.  Placement by atomic cursor bumps, then
// every bucket's segment is put back in input order (k_bucket_order on the
// element indices), then the ids are gathered.
__global__ void k_sbb_place(int64_t n, const int64_t* __restrict__ buckets, unsigned long long* __restrict__ cursor,
                            int32_t* __restrict__ slot_j) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x)
        slot_j[atomicAdd(cursor + buckets[j], 1ull)] = int32_t(j);
}

__global__ void k_sbb_counts(int64_t P, const int64_t* __restrict__ start, const int64_t* __restrict__ cursor,
                             int64_t* __restrict__ cnt) {
    for (int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; b < P; b += int64_t(gridDim.x) * blockDim.x)
        cnt[b] = cursor[b] - start[b];
}

// one warp per bucket: out_ids over the bucket's (now ordered) segment
__global__ void k_sbb_gather(int64_t P, const int64_t* __restrict__ start, const int64_t* __restrict__ cnt,
                             const int32_t* __restrict__ slot_j, const int64_t* __restrict__ orig_ids,
                             int64_t* __restrict__ out_ids) {
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t b = blockIdx.x * int64_t(blockDim.x >> 5) + warp_id(); b < P; b += warps) {
        const int64_t s0 = start[b], c = cnt[b];
        for (int64_t k = lane_id(); k < c; k += 32) out_ids[s0 + k] = orig_ids[slot_j[s0 + k]];
    }
}

int levels_for(int wp, int hp) {
    int m = wp > hp ? wp : hp, lv = 0;
    while ((1 << lv) < m) lv++;
    return lv;
}

struct BuildWs {
    int32_t *lin, *cnt, *mrank, *mcnt, *mstart, *cursor, *slot_pid, *big_list, *big_n;
    void* scan;
};

BuildWs carve_build(Carver& c, int64_t n, int64_t P) {
    BuildWs w;
    w.lin = c.take<int32_t>(n > 0 ? n : 1);
    w.cnt = c.take<int32_t>(P);
    w.mrank = c.take<int32_t>(P);
    w.mcnt = c.take<int32_t>(P);
    w.mstart = c.take<int32_t>(P + 1);
    w.cursor = c.take<int32_t>(P);
    w.slot_pid = c.take<int32_t>(n > 0 ? n : 1);
    w.big_list = c.take<int32_t>(P);
    w.big_n = c.take<int32_t>(1);
    w.scan = c.take<char>(scan_workspace_bytes(P + 1));
    return w;
}

}  // namespace
}  // namespace hp

using namespace hp;

extern "C" int hp_build_workspace_bytes(int64_t n, int64_t padded_w, int64_t padded_h, size_t* bytes) {
    Carver c(nullptr, 0);
    carve_build(c, n, padded_w * padded_h);
    *bytes = c.used + 256;
    return HP_OK;
}

extern "C" int hp_build(const double* positions, int64_t n, const hp_camera* cam, int64_t pad,
                        int64_t* table_start, int64_t* table_count, int64_t* reordered_ids,
                        double* slot_x, double* slot_y, double* slot_z, hp_query_layout layout,
                        int64_t* n_in, void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    if (!cam || pad < 0 || n < 0) {
        set_error("hp_build: invalid arguments");
        return HP_EINVAL;
    }
    const int64_t wp = cam->width + 2 * pad, hp_ = cam->height + 2 * pad;
    if (wp > 0xFFFF || hp_ > 0xFFFF) {
        set_error("padded image exceeds 16-bit pixel coordinates");
        return HP_EINVAL;
    }
    if (n >= (int64_t(1) << 31)) {
        set_error("hp_build: point count must be below 2^31");
        return HP_EINVAL;
    }
    const int64_t P = wp * hp_;
    if (P >= (int64_t(1) << 31)) {  // bucket ids, row pointers and scans are int32
        set_error("hp_build: padded grid of %lld pixels must be below 2^31", (long long)P);
        return HP_EINVAL;
    }
    Carver c(workspace, workspace_bytes);
    BuildWs w = carve_build(c, n, P);
    if (!c.ok()) {
        set_error("hp_build: workspace too small (%zu < %zu)", workspace_bytes, c.used);
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CamDev cd;
    for (int k = 0; k < 3; k++) {
        cd.o[k] = cam->origin[k];
        cd.r[k] = cam->right[k];
        cd.u[k] = cam->up[k];
        cd.f[k] = cam->forward[k];
    }
    cd.focal = cam->focal_length;
    cd.pw = cam->pixel_width;
    cd.ph = cam->pixel_height;
    cd.half_w = 0.5 * double(cam->width);
    cd.half_h = 0.5 * double(cam->height);

    TimedSpan ts("hp_build", s);
    if (cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * P, s) != cudaSuccess ||
        cudaMemsetAsync(w.big_n, 0, sizeof(int32_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_build memset");
    if (n > 0) {
        k_project<<<grid_for(n, kProjThreads, 148 * 16), kProjThreads, 0, s>>>(positions, n, cd, int(pad),
                                                                               int(wp), int(hp_), w.lin, w.cnt);
        HP_CHECK_LAUNCH("k_project");
    }
    const int levels = levels_for(int(wp), int(hp_));
    k_morton_permute<<<grid_for(P, 256), 256, 0, s>>>(int(wp), int(hp_), levels, w.cnt, w.mrank, w.mcnt);
    HP_CHECK_LAUNCH("k_morton_permute");
    HP_TRY(exclusive_scan_i32(w.mcnt, w.mstart, P, w.scan, s));
    HP_TRY(exclusive_scan_i32(w.cnt, layout.row_ptr, P, w.scan, s));
    k_tables<<<grid_for(P, 256), 256, 0, s>>>(P, w.cnt, w.mrank, w.mstart, table_start, table_count,
                                             w.cursor, layout.row_ptr, n_in);
    HP_CHECK_LAUNCH("k_tables");
    if (n > 0) {
        k_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, w.lin, w.cursor, w.slot_pid);
        HP_CHECK_LAUNCH("k_scatter");
        k_bucket_order<<<grid_for(P, 128), 128, 0, s>>>(P, table_start, table_count, w.slot_pid,
                                                         w.big_list, w.big_n);
        HP_CHECK_LAUNCH("k_bucket_order");
        k_big_bucket_order<<<148, 512, 0, s>>>(table_start, table_count, w.slot_pid, w.big_list, w.big_n);
        HP_CHECK_LAUNCH("k_big_bucket_order");
        k_gather<<<grid_for(n, 256), 256, 0, s>>>(n, n_in, positions, w.slot_pid, w.lin, table_start,
                                                 cam->origin[0], cam->origin[1], cam->origin[2],
                                                 reordered_ids, slot_x, slot_y, slot_z, layout);
        HP_CHECK_LAUNCH("k_gather");
    }
    return HP_OK;
}

// Layout-only build (the query layout of the rows a frame's rays can reach,
// no reference HashIndex arrays): every placed point goes straight to its
// row-major slot (warp-aggregated cursor bumps, the order inside a pixel is
// the atomics' -- the query ranks by (t, id), so results do not depend on it).
// (slot -> point by the scatter of k_scatter, then this gather: the layout's
// writes stay coalesced, the reads of the points are the random ones)
__global__ void k_gather_layout(const int64_t* __restrict__ n_in_dev, const double* __restrict__ xyz,
                                const int32_t* __restrict__ slot_pid, double o0, double o1, double o2,
                                hp_query_layout L) {
    const int64_t n_in = *n_in_dev;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n_in; k += int64_t(gridDim.x) * blockDim.x) {
        const int32_t id = slot_pid[k];
        const double rx = hp::dsub(xyz[3 * int64_t(id)], o0), ry = hp::dsub(xyz[3 * int64_t(id) + 1], o1),
                     rz = hp::dsub(xyz[3 * int64_t(id) + 2], o2);
        L.rel_x[k] = rx;
        L.rel_y[k] = ry;
        L.rel_z[k] = rz;
        L.point_id[k] = id;
        reinterpret_cast<float4*>(L.relf)[k] = filter_point(rx, ry, rz);
        store_rel4(L.rel4, k, rx, ry, rz, id);
    }
}

__global__ void k_layout_n_in(const int32_t* __restrict__ row_ptr, int64_t P, int64_t* __restrict__ n_in) {
    *n_in = row_ptr[P];
}

extern "C" int hp_build_layout_workspace_bytes(int64_t n, int64_t padded_w, int64_t padded_h, size_t* bytes) {
    const int64_t P = padded_w * padded_h;
    const int64_t nn = n > 0 ? n : 1;
    *bytes = 4 * 256 + 2 * ((sizeof(int32_t) * nn + 255) & ~size_t(255)) +
             2 * ((sizeof(int32_t) * (P + 1) + 255) & ~size_t(255)) + scan_workspace_bytes(P + 1) + 256;
    return HP_OK;
}

extern "C" int hp_build_layout(const double* positions, int64_t n, const hp_camera* cam, int64_t pad, int64_t row0,
                               int64_t row1, hp_query_layout layout, int64_t* n_in, void* workspace,
                               size_t workspace_bytes, hp_stream_t stream) {
    if (!cam || pad < 0 || n < 0) {
        set_error("hp_build_layout: invalid arguments");
        return HP_EINVAL;
    }
    const int64_t wp = cam->width + 2 * pad, hp_ = cam->height + 2 * pad;
    if (wp > 0xFFFF || hp_ > 0xFFFF) {
        set_error("padded image exceeds 16-bit pixel coordinates");
        return HP_EINVAL;
    }
    if (n >= (int64_t(1) << 31)) {
        set_error("hp_build_layout: point count must be below 2^31");
        return HP_EINVAL;
    }
    const int64_t P = wp * hp_;
    if (P >= (int64_t(1) << 31)) {
        set_error("hp_build_layout: padded grid of %lld pixels must be below 2^31", (long long)P);
        return HP_EINVAL;
    }
    Carver c(workspace, workspace_bytes);
    int32_t* lin = c.take<int32_t>(n > 0 ? n : 1);
    int32_t* slot_pid = c.take<int32_t>(n > 0 ? n : 1);
    int32_t* cnt = c.take<int32_t>(P + 1);
    int32_t* cursor = c.take<int32_t>(P + 1);
    void* scan = c.take<char>(scan_workspace_bytes(P + 1));
    if (!c.ok()) {
        set_error("hp_build_layout: workspace too small");
        return HP_ESPACE;
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CamDev cd;
    for (int k = 0; k < 3; k++) {
        cd.o[k] = cam->origin[k];
        cd.r[k] = cam->right[k];
        cd.u[k] = cam->up[k];
        cd.f[k] = cam->forward[k];
    }
    cd.focal = cam->focal_length;
    cd.pw = cam->pixel_width;
    cd.ph = cam->pixel_height;
    cd.half_w = 0.5 * double(cam->width);
    cd.half_h = 0.5 * double(cam->height);
    const int r0 = int(row0 < 0 ? 0 : (row0 > hp_ ? hp_ : row0));
    const int r1 = int(row1 <= 0 || row1 > hp_ ? hp_ : row1);
    TimedSpan ts("hp_build", s);
    if (cudaMemsetAsync(cnt, 0, sizeof(int32_t) * P, s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_build_layout memset");
    if (n > 0) {
        k_project<<<grid_for(n, kProjThreads, 148 * 16), kProjThreads, 0, s>>>(positions, n, cd, int(pad), int(wp),
                                                                               int(hp_), lin, cnt, r0, r1);
        HP_CHECK_LAUNCH("k_project");
    }
    HP_TRY(exclusive_scan_i32(cnt, layout.row_ptr, P, scan, s));
    if (cudaMemcpyAsync(cursor, layout.row_ptr, sizeof(int32_t) * P, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_build_layout copy");
    k_layout_n_in<<<1, 1, 0, s>>>(layout.row_ptr, P, n_in);
    HP_CHECK_LAUNCH("k_layout_n_in");
    if (n > 0) {
        k_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, lin, cursor, slot_pid);
        HP_CHECK_LAUNCH("k_scatter");
        k_gather_layout<<<grid_for(n, 256), 256, 0, s>>>(n_in, positions, slot_pid, cam->origin[0], cam->origin[1],
                                                         cam->origin[2], layout);
        HP_CHECK_LAUNCH("k_gather_layout");
    }
    return HP_OK;
}

extern "C" int hp_layout_workspace_bytes(int64_t n_in, int64_t padded_w, int64_t padded_h, size_t* bytes) {
    const int64_t P = padded_w * padded_h;
    *bytes = ((sizeof(int32_t) * P + 255) & ~size_t(255)) + scan_workspace_bytes(P + 1) + 512;
    (void)n_in;
    return HP_OK;
}

extern "C" int hp_layout_from_table(const int64_t* table_start, const int64_t* table_count,
                                    const double* slot_x, const double* slot_y, const double* slot_z,
                                    const int64_t* slot_ids, int64_t n_in, int64_t padded_w,
                                    int64_t padded_h, const double* origin_host, hp_query_layout layout,
                                    void* workspace, size_t workspace_bytes, hp_stream_t stream) {
    const int64_t P = padded_w * padded_h;
    if (padded_w < 0 || padded_h < 0 || n_in < 0 || P >= (int64_t(1) << 31) || n_in >= (int64_t(1) << 31)) {
        set_error("hp_layout_from_table: padded grid and point count must be below 2^31");
        return HP_EINVAL;
    }
    Carver c(workspace, workspace_bytes);
    int32_t* cnt = c.take<int32_t>(P);
    void* scan = c.take<char>(scan_workspace_bytes(P + 1));
    if (!c.ok()) {
        set_error("hp_layout_from_table: workspace too small");
        return HP_ESPACE;
    }
    (void)n_in;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    k_layout_counts<<<grid_for(P, 256), 256, 0, s>>>(P, table_count, cnt);
    HP_CHECK_LAUNCH("k_layout_counts");
    HP_TRY(exclusive_scan_i32(cnt, layout.row_ptr, P, scan, s));
    k_layout_fill<<<grid_for(P * 32, 256), 256, 0, s>>>(P, table_start, table_count, slot_x, slot_y, slot_z,
                                                        slot_ids, origin_host[0], origin_host[1],
                                                        origin_host[2], layout);
    HP_CHECK_LAUNCH("k_layout_fill");
    return HP_OK;
}

extern "C" int hp_scatter_by_bucket_workspace_bytes(int64_t n, int64_t n_buckets, int64_t n_out, size_t* bytes) {
    Carver c(nullptr, 0);
    c.take<int64_t>(n_buckets > 0 ? n_buckets : 1);
    c.take<int64_t>(n_buckets > 0 ? n_buckets : 1);
    c.take<int32_t>(n_out > 0 ? n_out : 1);
    c.take<int32_t>(n_buckets > 0 ? n_buckets : 1);
    c.take<int32_t>(1);
    *bytes = c.used + 256;
    (void)n;
    return HP_OK;
}

extern "C" int hp_scatter_by_bucket(const int64_t* buckets, const int64_t* orig_ids, int64_t n, int64_t* cursor,
                                    int64_t n_buckets, int64_t* out_ids, int64_t n_out, void* workspace,
                                    size_t workspace_bytes, hp_stream_t stream) {
    if (n < 0 || n_buckets < 0 || n_out < 0 || n >= (int64_t(1) << 31) || n_out >= (int64_t(1) << 31)) {
        set_error("hp_scatter_by_bucket: invalid sizes");
        return HP_EINVAL;
    }
    Carver c(workspace, workspace_bytes);
    int64_t* start = c.take<int64_t>(n_buckets > 0 ? n_buckets : 1);
    int64_t* cnt = c.take<int64_t>(n_buckets > 0 ? n_buckets : 1);
    int32_t* slot_j = c.take<int32_t>(n_out > 0 ? n_out : 1);
    int32_t* big_list = c.take<int32_t>(n_buckets > 0 ? n_buckets : 1);
    int32_t* big_n = c.take<int32_t>(1);
    if (!c.ok()) {
        set_error("hp_scatter_by_bucket: workspace too small");
        return HP_ESPACE;
    }
    if (n == 0) return HP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(start, cursor, size_t(n_buckets) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess ||
        cudaMemsetAsync(big_n, 0, sizeof(int32_t), s) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "hp_scatter_by_bucket copy");
    k_sbb_place<<<grid_for(n, 256), 256, 0, s>>>(n, buckets, reinterpret_cast<unsigned long long*>(cursor), slot_j);
    HP_CHECK_LAUNCH("k_sbb_place");
    k_sbb_counts<<<grid_for(n_buckets, 256), 256, 0, s>>>(n_buckets, start, cursor, cnt);
    HP_CHECK_LAUNCH("k_sbb_counts");
    k_bucket_order<<<grid_for(n_buckets, 256), 256, 0, s>>>(n_buckets, start, cnt, slot_j, big_list, big_n);
    HP_CHECK_LAUNCH("k_bucket_order");
    k_big_bucket_order<<<device_sms() * 2, 512, 0, s>>>(start, cnt, slot_j, big_list, big_n);
    HP_CHECK_LAUNCH("k_big_bucket_order");
    k_sbb_gather<<<grid_for(n_buckets * 32, 256), 256, 0, s>>>(n_buckets, start, cnt, slot_j, orig_ids, out_ids);
    HP_CHECK_LAUNCH("k_sbb_gather");
    return HP_OK;
}
