// hp_sortnet.cuh — CTA-wide all-ascending bitonic sorting network.
//
// Every comparator puts the minimum at the lower index, so a non-power-of-two
// array behaves as if padded with +inf: comparators whose upper index is out
// of range are no-ops and are skipped.  Used for the rare large segments
// (pixel buckets with many points, rays with more candidates than fit in
// shared memory); the common path sorts in shared memory elsewhere.
#pragma once

namespace hp {

// less(a, b): element at index a orders before element at index b.
// swap(a, b): exchange elements a and b.  Must be called by all threads of
// the block; indices are segment-relative.
template <class Less, class Swap>
__device__ void block_bitonic_sort(int64_t n, Less less, Swap swap) {
    if (n < 2) return;
    int64_t np2 = 1;
    while (np2 < n) np2 <<= 1;
    const int64_t half = np2 >> 1;
    for (int64_t k = 2; k <= np2; k <<= 1) {
        const int64_t hk = k >> 1;
        for (int64_t t = threadIdx.x; t < half; t += blockDim.x) {  // mirror step
            const int64_t blk = (t / hk) * k, o = t % hk;
            const int64_t a = blk + o, b = blk + k - 1 - o;
            if (b < n && less(b, a)) swap(a, b);
        }
        __syncthreads();
        for (int64_t j = hk >> 1; j > 0; j >>= 1) {                  // half cleaners
            for (int64_t t = threadIdx.x; t < half; t += blockDim.x) {
                const int64_t a = (t / j) * 2 * j + (t % j), b = a + j;
                if (b < n && less(b, a)) swap(a, b);
            }
            __syncthreads();
        }
    }
}

}  // namespace hp
