// hp_common.cu — error state, launch accounting and the device-wide exclusive
// scan used for CSR offsets, Morton-order table starts and row pointers.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>

#include "hp_common.cuh"

namespace hp {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
    set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
    return HP_ECUDA;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Per-device launch facts: the SM count, and per (kernel, device) the
// max-dynamic-shared-memory attribute (set once) and the resident CTAs per
// SM at the given block size / shared memory.  Function attributes apply per
// device, so a process that moves to another GPU configures it there too.
namespace {
std::mutex g_dev_mu;
std::map<int, int> g_sms;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;
}  // namespace

int device_sms() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return 148;
    }
    std::lock_guard<std::mutex> lk(g_dev_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = 148;
    }
    g_sms[dev] = n;
    return n;
}

int kernel_occupancy(const void* fn, int threads, size_t smem) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    const auto key = std::make_tuple(fn, dev, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute");
    }
    if (smem > 0) {  // the whole unified L1 / shared array as shared memory (occupancy counts on it)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute carveout");
    }
    int n = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
    if (n < 1) {
        set_error("kernel does not fit one CTA per SM (%d threads, %zu B shared memory)", threads, smem);
        return HP_ECUDA;
    }
    g_occ[key] = n;
    return n;
}

// ------------------------------------------------------------------ timing
namespace {
struct Pending {
    std::string name;
    cudaEvent_t a, b;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
std::vector<Pending> g_open;  // begun, not ended (per nesting level)
cudaEvent_t take_event() {
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
}  // namespace

void timing_begin(const char* name, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing) return;
    Pending p{name, take_event(), take_event()};
    cudaEventRecord(p.a, s);
    g_open.push_back(p);
}

void timing_end(cudaStream_t s) {
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing || g_open.empty()) return;
    Pending p = g_open.back();
    g_open.pop_back();
    cudaEventRecord(p.b, s);
    g_pending.push_back(p);
}

// ------------------------------------------------------------------ scan
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int64_t kScanTile = int64_t(kScanThreads) * kScanItems;

template <class In>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums(const In* __restrict__ in, int64_t n,
                                                               int64_t* __restrict__ sums) {
    __shared__ int64_t sh[kScanThreads / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    int64_t acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++)
        if (base + k < n) acc += static_cast<int64_t>(in[base + k]);
    int64_t total;
    block_excl_scan<int64_t>(acc, sh, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// one block: exclusive scan of the tile sums (sequential chunks per thread)
__global__ void __launch_bounds__(1024) scan_sums(int64_t* __restrict__ sums, int64_t tiles) {
    __shared__ int64_t sh[1024 / 32 + 1];
    const int64_t per = (tiles + blockDim.x - 1) / blockDim.x;
    const int64_t lo = int64_t(threadIdx.x) * per;
    const int64_t hi = lo + per < tiles ? lo + per : tiles;
    int64_t acc = 0;
    for (int64_t i = lo; i < hi; i++) acc += sums[i];
    int64_t total;
    int64_t run = block_excl_scan<int64_t>(acc, sh, &total);
    for (int64_t i = lo; i < hi; i++) {
        int64_t v = sums[i];
        sums[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) sums[tiles] = total;
}

template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) scan_tiles(const In* in, Out* out, int64_t n,
                                                           const int64_t* __restrict__ sums) {
    __shared__ int64_t sh[kScanThreads / 32 + 1];
    const int64_t base = int64_t(blockIdx.x) * kScanTile + int64_t(threadIdx.x) * kScanItems;
    int64_t v[kScanItems];
    int64_t acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        v[k] = base + k < n ? static_cast<int64_t>(in[base + k]) : 0;
        acc += v[k];
    }
    int64_t total;
    int64_t run = block_excl_scan<int64_t>(acc, sh, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) out[base + k] = static_cast<Out>(run);
        run += v[k];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = static_cast<Out>(sums[gridDim.x]);
}

size_t scan_workspace_bytes(int64_t n) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles < 1) tiles = 1;
    return size_t(tiles + 1) * sizeof(int64_t) + 256;
}

template <class In, class Out>
static int scan_impl(const In* in, Out* out, int64_t n, void* ws, cudaStream_t s) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles < 1) tiles = 1;
    int64_t* sums = static_cast<int64_t*>(ws);
    scan_tile_sums<In><<<unsigned(tiles), kScanThreads, 0, s>>>(in, n, sums);
    HP_CHECK_LAUNCH("scan_tile_sums");
    scan_sums<<<1, 1024, 0, s>>>(sums, tiles);
    HP_CHECK_LAUNCH("scan_sums");
    scan_tiles<In, Out><<<unsigned(tiles), kScanThreads, 0, s>>>(in, out, n, sums);
    HP_CHECK_LAUNCH("scan_tiles");
    return HP_OK;
}

int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, void* ws, cudaStream_t s) {
    return scan_impl<int64_t, int64_t>(in, out, n, ws, s);
}
int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* ws, cudaStream_t s) {
    return scan_impl<int32_t, int32_t>(in, out, n, ws, s);
}
int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, void* ws,
                              cudaStream_t s) {
    return scan_impl<int32_t, int64_t>(in, out, n, ws, s);
}

}  // namespace hp

extern "C" int hp_timing_enable(int on) {
    std::lock_guard<std::mutex> lk(hp::g_tmu);
    hp::g_timing = on != 0;
    return HP_OK;
}

// Synchronises on the recorded events and returns, per kernel name, the summed
// milliseconds and launch counts ("name1\nname2\n..." in names).  Clears.
extern "C" int hp_timing_collect(char* names, int names_len, double* ms, int64_t* counts, int max_entries,
                                 int* n_entries) {
    std::lock_guard<std::mutex> lk(hp::g_tmu);
    std::vector<std::string> keys;
    std::vector<double> sums;
    std::vector<int64_t> cnts;
    for (auto& p : hp::g_pending) {
        cudaEventSynchronize(p.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, p.a, p.b);
        size_t k = 0;
        while (k < keys.size() && keys[k] != p.name) k++;
        if (k == keys.size()) {
            keys.push_back(p.name);
            sums.push_back(0.0);
            cnts.push_back(0);
        }
        sums[k] += t;
        cnts[k] += 1;
        hp::g_pool.push_back(p.a);
        hp::g_pool.push_back(p.b);
    }
    hp::g_pending.clear();
    std::string joined;
    int n = 0;
    for (size_t k = 0; k < keys.size() && n < max_entries; k++, n++) {
        ms[n] = sums[k];
        counts[n] = cnts[k];
        joined += keys[k];
        joined += "\n";
    }
    if (names && names_len > 0) {
        strncpy(names, joined.c_str(), size_t(names_len - 1));
        names[names_len - 1] = 0;
    }
    *n_entries = n;
    return HP_OK;
}

namespace hp {
namespace {
std::mutex g_chk_mu;
std::vector<CheckReader>& check_readers() {
    static std::vector<CheckReader> v;
    return v;
}
}  // namespace
int register_check_reader(CheckReader f) {
    std::lock_guard<std::mutex> lk(g_chk_mu);
    check_readers().push_back(f);
    return int(check_readers().size());
}
}  // namespace hp

// Checked build: the source lines of the first failing HP_ASSERT of each
// translation unit (0 = none), up to max_out of them; returns how many
// translation units report a failure (always 0 in the normal build).
extern "C" int hp_check_failures(int64_t* lines, int max_out, int reset) {
    std::lock_guard<std::mutex> lk(hp::g_chk_mu);
    int n = 0;
    for (auto f : hp::check_readers()) {
        unsigned long long v = 0;
        if (f(&v, reset) != 0) return hp::cuda_status(cudaGetLastError(), "hp_check_failures");
        if (v) {
            if (n < max_out && lines) lines[n] = int64_t(v);
            n++;
        }
    }
    return n;
}

extern "C" const char* hp_last_error(void) { return hp::g_err; }
extern "C" int hp_version(void) { return 1; }
extern "C" int64_t hp_launch_count(void) { return hp::g_launches.load(); }
