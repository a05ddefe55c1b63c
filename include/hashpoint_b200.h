/*
 * hashpoint_b200.h — C ABI of the B200-native HashPoint hot path.
 *
 * Drop-in boundary for the reference's operator layer.  All
 * array arguments are DEVICE pointers (cudaMalloc / torch CUDA tensors),
 * C-contiguous, in the reference's dtypes (int64 ids/offsets/tables, float64
 * coordinates and values).  Sizes are element counts.  Every function returns
 * 0 on success or a negative HP_E* code; hp_last_error() returns a
 * thread-local message for the last failure.  Functions are stateless and
 * enqueue work on `stream` (a cudaStream_t); they never synchronise the device
 * except where stated.  Scratch comes from a caller-provided workspace whose
 * size the matching *_workspace_bytes function reports.
 *
 * Reference interfaces replaced (reference = /root/reference/pkg/src/hashpoint):
 *   hp_build            hash_index.build            hash_index.py:151-190
 *   hp_scatter_by_bucket _kernels.scatter_by_bucket  _kernels.py:76-83
 *                       + _kernels.scatter_by_bucket  _kernels.py:76-83
 *                       + rasterize_points / morton_codes hash_index.py:81-112
 *   hp_layout_from_table (internal re-layout of a HashIndex built elsewhere;
 *                       consumes the arrays of HashIndex hash_index.py:115-148)
 *   hp_query_count /    _kernels.hash_query_batch   _kernels.py:86-157
 *   hp_query_fill         (+ _cone_test :22-36, _canonical_sort :39-73);
 *                       two-phase because Q is unknown before the call
 *                       (the reference grows its buffers, :141-151)
 *   hp_head_count /     hash_query_batch -> sample_batch chained as in
 *   hp_head_sort          renderer.py:119-124 (the sampler's heads only)
 *   hp_sample_run /     _kernels.sample_batch        _kernels.py:552-700
 *   hp_sample_emit        (two-phase for the same reason; R unknown)
 *   hp_primary_surface  derived: first retained candidate per ray
 *   hp_ray_grid         geometry.ray_grid            geometry.py:289-306
 *   hp_radius_slopes    geometry.radius_slopes       geometry.py:249-260
 *   hp_render           renderer.render_volume / render_knp renderer.py:138-185
 *   hp_pointnerf_*      (no reference symbol) the Point-NeRF aggregation MLP the
 *                       paper integrates with, cfg5
 */
#ifndef HASHPOINT_B200_H
#define HASHPOINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HP_OK 0
#define HP_EINVAL (-1)  /* invalid argument (the reference raises ValueError) */
#define HP_ECUDA (-2)   /* CUDA runtime error (RuntimeError) */
#define HP_ESPACE (-3)  /* workspace too small */

typedef void* hp_stream_t; /* cudaStream_t */

/* Pinhole camera (reference geometry.py:50-134). Host struct, passed by pointer. */
typedef struct {
    double origin[3];
    double right[3];
    double up[3];
    double forward[3];
    double focal_length;
    double pixel_width;
    double pixel_height;
    int64_t width;
    int64_t height;
} hp_camera;

/* Query layout: the index's points re-laid out row-major by padded pixel
 * (within a pixel: ascending original id, as in the reference's slots), with
 * coordinates pre-shifted by the camera origin.  A kernel row of s pixels is
 * then ONE contiguous slot range.  Device arrays; caller-allocated:
 * row_ptr[P+1], rel_x/rel_y/rel_z/point_id[N_in], relf[4*N_in] (capacity n
 * for hp_build).  relf holds (x, y, z, e) in float32 for the filter: the
 * rounded coordinates and the point's error budget e = 2^-18 * |p|_1.
 * rel4[4*N_in] holds the same point as one 32-byte record (x, y, z, id as
 * int64 bits) so that a single sector gather gives the exact coordinates of
 * a slot (the head sort recomputes t / dist from it). */
typedef struct {
    int32_t* row_ptr;
    double* rel_x;
    double* rel_y;
    double* rel_z;
    int32_t* point_id;
    float* relf;
    double* rel4;
} hp_query_layout;

typedef struct {
    int32_t k_neighbors; /* K >= 1 (device limit HP_MAX_K) */
    int32_t eps_mode;    /* 1: keep w >= eps; 0: tau mode */
    int32_t want_color;  /* 1: colors != NULL, emit r_color */
    int32_t exact_t_end; /* 1: t_end over all candidates (reference semantics);
                            0: transmittance at the exit of retention */
    double beta2;        /* beta*beta, computed by the caller as in sampler.py:215 */
    double gamma;
    double eps;
    double tau_min;
    int32_t emit_knn;    /* 1: also emit each retained sample's K neighbour point
                            ids and blend weights (hp_sample_emit*: r_knn_id /
                            r_knn_w [R, k_neighbors]; the K nearest of
                            _kernels.py:603-620 and the weights of its colour
                            blend :622-656, w_b = (1/d_b) / sum(1/d); coincident
                            points 1/nz; -1 / 0 past the pool size) */
    int32_t reserved;
} hp_sampler_params;

#define HP_MAX_K 256

const char* hp_last_error(void);
int hp_version(void);

/* ---------------- build ---------------- */
int hp_build_workspace_bytes(int64_t n, int64_t padded_w, int64_t padded_h, size_t* bytes);
/* positions: float64 [n,3].  Outputs: table_start/table_count int64 [P];
 * reordered_ids int64, slot_x/y/z float64 with capacity n; layout (capacity n);
 * n_in: device int64 scalar receiving N_in.  Errors: padded size > 0xFFFF
 * ("padded image exceeds 16-bit pixel coordinates"), n >= 2^31. */
int hp_build(const double* positions, int64_t n, const hp_camera* cam, int64_t pad,
             int64_t* table_start, int64_t* table_count, int64_t* reordered_ids,
             double* slot_x, double* slot_y, double* slot_z, hp_query_layout layout,
             int64_t* n_in, void* workspace, size_t workspace_bytes, hp_stream_t stream);

/* The query layout alone (no reference HashIndex arrays) for the padded rows
 * [row0, row1) (row1 <= 0: all): what a frame that only queries needs (the
 * points outside the rows are left out; inside a pixel the order is
 * arbitrary -- the query ranks matches by (t, id)).  n_in [1] (device) = the
 * placed points.  Rays of image rows [a, b) reach padded rows [a, b + 2 pad). */
int hp_build_layout_workspace_bytes(int64_t n, int64_t padded_w, int64_t padded_h, size_t* bytes);
int hp_build_layout(const double* positions, int64_t n, const hp_camera* cam, int64_t pad, int64_t row0,
                    int64_t row1, hp_query_layout layout, int64_t* n_in, void* workspace, size_t workspace_bytes,
                    hp_stream_t stream);

/* The reference's counting-sort placement operator on its own
 * (_kernels.scatter_by_bucket, _kernels.py:76-83): for j in input order,
 * out_ids[cursor[buckets[j]]++] = orig_ids[j].  buckets / orig_ids int64 [n],
 * cursor int64 [n_buckets] (updated in place, as the reference), out_ids
 * int64 [n_out] (only the placed positions are written).  The buckets'
 * destination ranges must not overlap (cursor = an exclusive scan of the
 * counts, as hash_index.build passes it); the caller checks ranges. */
int hp_scatter_by_bucket_workspace_bytes(int64_t n, int64_t n_buckets, int64_t n_out, size_t* bytes);
int hp_scatter_by_bucket(const int64_t* buckets, const int64_t* orig_ids, int64_t n, int64_t* cursor,
                         int64_t n_buckets, int64_t* out_ids, int64_t n_out, void* workspace,
                         size_t workspace_bytes, hp_stream_t stream);

int hp_layout_workspace_bytes(int64_t n_in, int64_t padded_w, int64_t padded_h, size_t* bytes);
int hp_layout_from_table(const int64_t* table_start, const int64_t* table_count,
                         const double* slot_x, const double* slot_y, const double* slot_z,
                         const int64_t* slot_ids, int64_t n_in, int64_t padded_w,
                         int64_t padded_h, const double* origin_host, hp_query_layout layout,
                         void* workspace, size_t workspace_bytes, hp_stream_t stream);

/* ---------------- host helpers ---------------- */
/* Per-ray search-radius slopes on host threads (replaces the vectorised
 * geometry.radius_slopes, reference geometry.py:249-260): same expression
 * order and libm calls as numpy, bit-identical; pixels int64 [m,2] with
 * element stride pixel_stride between rays, or NULL for the camera's ray
 * grid (ray k = pixel (k % width, k / width)); slopes float64 [m] (host). */
int hp_radius_slopes_host(const hp_camera* cam, const int64_t* pixels, int64_t pixel_stride, int64_t m,
                          double kernel_radius, int approx, double* slopes, int threads);

/* The same slopes on the device (replaces geometry.radius_slopes,
 * geometry.py:249-260, bit-identical to numpy: glibc's hypot restated in
 * round-to-nearest): pixels int64 [m,2] on the device with element stride
 * pixel_stride, or NULL for rays row0 * width + k of the camera's ray grid;
 * slopes float64 [m] on the device. */
int hp_radius_slopes(const hp_camera* cam, int64_t row0, const int64_t* pixels, int64_t pixel_stride, int64_t m,
                     double kernel_radius, int approx, double* slopes, hp_stream_t stream);

/* Host -> device upload of PAGEABLE host memory (numpy arrays) through a
 * caller-provided pinned staging buffer of >= bytes: `threads` host threads
 * copy src into it in pieces of `piece` bytes (0: 2 MiB) and each piece's
 * cudaMemcpyAsync to dst is enqueued on `stream` as soon as it is staged.
 * Returns once every piece is enqueued; the staging buffer must stay
 * untouched until the stream has run the copies.  (Host plumbing of the
 * host-buffer entry points; no reference counterpart.) */
int hp_host_upload(void* dst, const void* src, size_t bytes, void* staging, size_t piece, int threads,
                   cudaStream_t stream);

/* The camera's ray grid on the device (replaces geometry.ray_grid,
 * geometry.py:289-306, bit-identical): rows [row0, row0 + rows) of the image,
 * ray k = (row0 * width + k) in row-major order.  dirs float64 [m,3] unit
 * directions through the pixel centres; pixels int64 [m,2] (u, v) or NULL;
 * t_near / t_far [m] filled with the given values, or NULL.
 * m = rows * cam->width. */
int hp_ray_grid(const hp_camera* cam, int64_t row0, int64_t rows, double* dirs, int64_t* pixels,
                double t_near_value, double t_far_value, double* t_near, double* t_far,
                hp_stream_t stream);

/* ---------------- query ---------------- */
/* capacity: scratch slots for the unsorted matches (hp_query_count reports
 * the number it needs). */
int hp_query_workspace_bytes(int64_t m, int64_t pad, int64_t capacity, size_t* bytes);
/* Pass 1 (the streaming pass).  cam: the index camera (host struct; NULL
 * tests every pixel of the s x s window, otherwise only pixels whose
 * directions can lie inside the ray's cone -- same result, fewer tests).
 * pixels: int64 [m,2] (u, v) with element stride pixel_stride between rays (2
 * for an (m,2) array); dirs float64 [m,3]; t_near/t_far/slopes [m].  Writes
 * probes/scanned [m] (int64, over the full window as the reference) and
 * offsets [m+1] (int64 CSR offsets; offsets[m] = Q); the accepted matches are
 * kept, unsorted, in the workspace (capacity slots).  No host round trip: if
 * the frame needs more than `capacity` slots nothing else is written and
 * offsets[m] = -(slots needed); the caller, which reads offsets[m] anyway to
 * allocate the outputs, grows the workspace and calls again. */
int hp_query_count(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                   int64_t pad,
                   const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                   const double* t_near, const double* t_far, const double* slopes, int64_t m,
                   int64_t* offsets, int64_t* probes, int64_t* scanned, int64_t capacity,
                   void* workspace, size_t workspace_bytes, hp_stream_t stream);
/* Heads (callers that only want samples; replaces hash_query_batch ->
 * sample_batch as chained by renderer.py:119-124): per ray, the head of its
 * matches in (t, id) order -- all of them when it has few, else the
 * smallest-t matches up to a cut near the `want`-th (want <= whole <= 1024:
 * rays of at most `whole` matches are sorted whole; with `rays`, whole up to
 * 4096 selects the long-head mode for rays 1024 do not cover, head_off
 * spaced for it) -- without the
 * full match list.  hp_head_count is the streaming pass (same arguments and
 * probes / scanned / offsets outputs as hp_query_count, offsets[m] = Q or
 * -(slots needed) when `capacity` is short); it keeps 8 bytes per match in
 * the workspace and writes head_off [m+1] = the exclusive scan of
 * min(q, 1024) (head_off[m] = the head arrays' capacity).  hp_head_sort
 * writes each ray's head at head_off[r]: head_t / head_dist float64,
 * head_ids int32 (same workspace and capacity), plen [m] = the head length,
 * facts [m] (as hp_query_fill's, over the head; -1 when unknown), and cut_t /
 * cut_d [m] = lower bounds of the t / dist of every match left out (+inf when
 * none).  hp_sample_run_prefix consumes them.  rays (int32 [n], or NULL for
 * all m rays): re-sort only these rays of the same count pass (e.g. with a
 * longer `want` for rays the sampler flagged); output i (head_off[i], plen[i],
 * facts[i], cuts[i]) then stands for ray rays[i].  sampler + head_u (both
 * or neither): the sampler's bound factors of every head entry (float, next
 * to head_t; -1 where not precomputed), which hp_sample_run_prefix then
 * multiplies instead of recomputing them (same results).  hp_head_sort may
 * be enqueued right after hp_head_count, before the caller has read
 * offsets[m]: the head arrays may then be sized by `capacity` (>= head_off[m]
 * whenever the count fit), and when the count ran short (offsets[m] < 0) it
 * writes empty heads and the caller re-runs both with the reported size. */
int hp_head_workspace_bytes(int64_t m, int64_t capacity, size_t* bytes);
int hp_head_count(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                  int64_t pad, const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                  const double* t_near, const double* t_far, const double* slopes, int64_t m,
                  int64_t* offsets, int64_t* head_off, int64_t* probes, int64_t* scanned,
                  int64_t capacity, void* workspace, size_t workspace_bytes, hp_stream_t stream);
int hp_head_sort(hp_query_layout layout, const double* dirs, const double* slopes, int64_t m,
                 const int64_t* offsets, const int32_t* rays, int64_t n, const int64_t* head_off, int32_t want,
                 int32_t whole, double* head_t, int32_t* head_ids, double* head_dist, int32_t* plen,
                 int32_t* facts, double* cut_t, double* cut_d, const hp_sampler_params* sampler, float* head_u,
                 int64_t capacity, void* workspace, size_t workspace_bytes, hp_stream_t stream);

/* Upper bounds of the match counts (the slots pass 1 will test per ray),
 * exclusive-scanned into bound_off [m+1] (bound_off[m] = the scratch pass 1
 * needs).  Lets a caller split a frame into ray chunks that fit memory.
 * workspace: >= hp_query_workspace_bytes(m, pad, 0). */
int hp_query_bounds(hp_query_layout layout, const hp_camera* cam, int64_t padded_w, int64_t padded_h,
                    int64_t pad, const int64_t* pixels, int64_t pixel_stride, const double* dirs,
                    const double* t_near, const double* t_far, const double* slopes, int64_t m,
                    int64_t* bound_off, void* workspace, size_t workspace_bytes, hp_stream_t stream);
/* Pass 2: sort each ray's matches by (t, id) from the workspace of pass 1
 * (same buffer, same capacity) into ids int64 [Q], t_proj / dist_perp
 * float64 [Q] (total = Q = offsets[m], host value).
 * facts (optional, int32 [m], NULL to skip; needs the query's slopes [m]):
 * per ray -1 (unknown) or, when every t / dist of the sorted segment is
 * finite with dist >= 0, the count #{dist <= slopes[r] * t_0}.  Passing them
 * to hp_sample_run for this exact CSR spares the sampler its full pass over
 * the CSR. */
int hp_query_fill(const int64_t* offsets, int64_t m, int64_t total, int64_t* ids, double* t_proj,
                  double* dist_perp, const double* slopes, int32_t* facts, int64_t capacity,
                  void* workspace, size_t workspace_bytes, hp_stream_t stream);

/* ---------------- sample ---------------- */
/* exact_capacity: slots for candidates evaluated exactly (udf/alpha/colour
 * scratch, one thread per candidate; the retained candidates are kept there,
 * compacted, between run and emit). */
int hp_sample_workspace_bytes(int64_t m, int64_t total, int64_t exact_capacity,
                              const hp_sampler_params* p, size_t* bytes);
/* Pass 1 over the query CSR (offsets [m+1], ids/t/dist [total], slopes [m],
 * colors float64 [n_colors,3] or NULL).  Writes t_end [m] and r_off [m+1]
 * (r_off[m] = R).  Retained candidates are kept in the workspace for emit.
 * No host round trip: if the exactly evaluated candidates exceed
 * exact_capacity, r_off[m] = -(slots needed) and the caller grows the
 * workspace and calls again.  query_facts: NULL, or the facts hp_query_fill
 * wrote for exactly this CSR and these slopes. */
int hp_sample_run(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                  const double* dist, int64_t total, int64_t exact_capacity, const double* slopes,
                  const int32_t* query_facts,
                  const hp_sampler_params* p, const double* colors, int64_t n_colors,
                  int64_t* r_off, double* t_end,
                  void* workspace, size_t workspace_bytes, hp_stream_t stream);
/* Pass 2: write the R retained candidates (R = r_off[m], host value) in ray
 * order: r_id int64, r_t/r_dist/r_udf/r_alpha/r_w float64 [R], r_color
 * float64 [R,3] (may be NULL without colors). */
int hp_sample_emit(const int64_t* offsets, int64_t m, const int64_t* ids, const double* t,
                   const double* dist, int64_t total, int64_t exact_capacity, const double* slopes,
                   const hp_sampler_params* p, const double* colors, int64_t n_colors,
                   const int64_t* r_off, int64_t R, int64_t* r_id,
                   double* r_t, double* r_dist, double* r_udf, double* r_alpha, double* r_w,
                   double* r_color, int64_t* r_knn_id, double* r_knn_w, void* workspace,
                   size_t workspace_bytes, hp_stream_t stream);

/* Prefix mode: the sampler over hp_head_sort's heads (offsets = the full
 * match counts from hp_head_count, query_facts = hp_head_sort's facts,
 * prefix = {head_off, plen, head_ids, head_t, head_dist, cut_t, cut_d}).  Results are those of hp_sample_run on the full CSR for
 * every ray not flagged; flagged [m+1] receives 1 for a ray whose work may
 * reach past its prefix (its r_off count is 0, its t_end NaN: run it through
 * the full path) and flagged[m] = the number of such rays. */
typedef struct hp_sample_prefix {
    const int64_t* start;  /* [m] */
    const int32_t* length; /* [m] */
    const int32_t* ids;
    const double* t;
    const double* dist;
    const double* cut_t;   /* [m] */
    const double* cut_d;   /* [m] */
    const float* u;        /* NULL, or hp_head_sort's head_u */
} hp_sample_prefix;
int hp_sample_run_prefix(const int64_t* offsets, int64_t m, const hp_sample_prefix* prefix,
                         int64_t exact_capacity, const double* slopes, const int32_t* query_facts,
                         const hp_sampler_params* p, const double* colors, int64_t n_colors,
                         int64_t* r_off, double* t_end, int32_t* flagged, void* workspace,
                         size_t workspace_bytes, hp_stream_t stream);
int hp_sample_emit_prefix(const int64_t* offsets, int64_t m, const hp_sample_prefix* prefix,
                          int64_t exact_capacity, const double* slopes, const hp_sampler_params* p,
                          const double* colors, int64_t n_colors, const int64_t* r_off, int64_t R,
                          int64_t* r_id, double* r_t, double* r_dist, double* r_udf, double* r_alpha,
                          double* r_w, double* r_color, int64_t* r_knn_id, double* r_knn_w, void* workspace,
                          size_t workspace_bytes, hp_stream_t stream);

/* Per-sample output arrays of a sampling pass (R rows each; r_color [R,3],
 * r_knn_id / r_knn_w [R,K], or NULL). */
typedef struct hp_sample_fields {
    int64_t* r_id;
    double* r_t;
    double* r_dist;
    double* r_udf;
    double* r_alpha;
    double* r_w;
    double* r_color;
    int64_t* r_knn_id;
    double* r_knn_w;
} hp_sample_fields;
/* Splice the samples of re-run rays into a pass's samples (the flagged rays
 * of hp_sample_run_prefix, which hold none there): output ray r (of m) takes
 * its rows from `sub` at s_off[pos[r]] when pos[r] >= 0, else from `main` at
 * r_off[r]; off_out [m+1] is the merged CSR (caller-computed).  k_neighbors:
 * the row width of the knn fields (0: none).  (Host plumbing of the head
 * path's second chance; no reference counterpart.) */
int hp_splice_samples(int64_t m, const int64_t* off_out, const int64_t* r_off, const int64_t* s_off,
                      const int64_t* pos, int32_t k_neighbors, const hp_sample_fields* main_rows,
                      const hp_sample_fields* sub_rows, const hp_sample_fields* out, hp_stream_t stream);

/* ---------------- Point-NeRF aggregation MLP (cfg5; bf16 on tcgen05) ----------------
 * The consumer of emit_knn.  No
 * reference implementation: parity vs an fp32 PyTorch
 * restatement (pointnerf.py).  hp_pointnerf_aggregate: per retained sample s
 * (R of them, k neighbours each, k a power of two <= 32), input rows
 * [feature (32 bf16) | sin/cos(2^l pi (p_i - x_s)), l < 4 | p_i - x_s | 1 | 0...]
 * (64), h1 = relu(W1 in), h2 = relu(W2 h1 + b2), g_s = sum_k w_sk h2 ->
 * g_out bf16 [R,128].  x_s = origin + r_t[s] * dirs[sample_ray[s]].
 * features: bf16 [n,32]; w1 bf16 [128,64]; w2 bf16 [128,128]; b2 f32 [128].
 * hp_pointnerf_head: out f32 [R,4] = (softplus, sigmoid x3) of
 * W4 relu(W3 g + b3) + b4; w3 bf16 [64,128], b3 f32 [64], w4 f32 [4,64],
 * b4 f32 [4].  Device pointers except origin_host (host double[3]). */
int hp_pointnerf_aggregate(const int64_t* knn_id, const double* knn_w, int64_t R, int32_t k,
                           const int32_t* sample_ray, const double* r_t, const double* dirs,
                           const double* origin_host, const double* positions, const uint16_t* features,
                           const uint16_t* w1, const uint16_t* w2, const float* b2, uint16_t* g_out,
                           hp_stream_t stream);
int hp_pointnerf_head(const uint16_t* g, int64_t R, const uint16_t* w3, const float* b3, const float* w4,
                      const float* b4, float* out, hp_stream_t stream);

/* ---------------- render (consumer of the samples) ---------------- */
/* Colour / depth of each ray's pixel from its retained samples (replaces the
 * per-ray loops of renderer.render_volume / render_knp, renderer.py:138-185).
 * mode 0 volume (uses r_alpha, r_color [R,3], t_far), 1 knp (uses r_dist,
 * r_id, point_colors [n,3], knp_k >= 1).  pixels int64 [m,2] (stride),
 * background: host double[3].  color [H,W,3] / depth [H,W] are written only
 * at the rays' pixels (the caller fills the blank image); several rays on
 * one pixel: the last ray wins.  owner: int32 [H*W] scratch. */
int hp_render(int mode, const int64_t* r_off, int64_t m, const int64_t* r_id, const double* r_t,
              const double* r_dist, const double* r_alpha, const double* r_color,
              const double* point_colors, const int64_t* pixels, int64_t pixel_stride,
              const double* t_far, int32_t knp_k, const double* background, int64_t width,
              int64_t height, int32_t* owner, double* color, double* depth, hp_stream_t stream);

/* out2[0] = offsets[m] (total), out2[1] = max_r (offsets[r+1] - offsets[r]).
 * Device int64[2]. */
int hp_csr_stats(const int64_t* offsets, int64_t m, int64_t* out2, hp_stream_t stream);

/* primary_id[r] = r_id[r_off[r]] or -1; primary_t[r] = r_t[r_off[r]] or NaN. */
int hp_primary_surface(const int64_t* r_off, int64_t m, const int64_t* r_id, const double* r_t,
                       int64_t* primary_id, double* primary_t, hp_stream_t stream);

/* Sampler path counters since the last reset (diagnostics; all zero unless
 * the library is built with -DHP_DEBUG_COUNTERS, e.g. `make DEBUG=1`):
 * [rays with candidates, fast-path rays, rays whose transmittance was proved 0,
 *  K-NN distance evaluations, candidates, bound factors evaluated, -, -]. */
int hp_sample_debug_counters(int64_t* out8, int reset);

/* Per-kernel CUDA-event timing on the launching stream (diagnostics and the
 * benchmark's roofline): enable, run, then collect per-name summed ms and
 * launch counts (names newline-separated); collect synchronises and clears. */
int hp_timing_enable(int on);
int hp_timing_collect(char* names, int names_len, double* ms, int64_t* counts, int max_entries,
                      int* n_entries);

/* Checked build (libhp_b200_checked.so, `make checked`): device-side
 * bounds / invariant checks record the source line of the first failure of
 * each translation unit; this returns how many report one (lines[] gets up
 * to max_out of them) and optionally clears them.  Always 0 in the normal
 * build. */
int hp_check_failures(int64_t* lines, int max_out, int reset);

/* Kernel launches issued by this library since load (for bench gpu_launches). */
int64_t hp_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
