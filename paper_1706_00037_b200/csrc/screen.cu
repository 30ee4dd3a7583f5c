// screen.cu — K-SCR: survivors = {k : f_k > floor(T)} in ascending slot order
// (Figure 2 "if xQx > Screening_value"; T(lambda) = Mean + lambda(Max - Mean)).
// T is formed on the host in binary64 (abi.cu); for integer f, f > T <=> f > floor(T).
// Two passes over f (8 B per solution): per-block counts, then an ordered block-local
// compaction at the block's prefix offset.  HBM-read bound; microseconds at K = 262144.
#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

constexpr int kScrThreads = 1024;
constexpr int kScrPer = 4;                        // consecutive elements per thread
constexpr int kScrChunk = kScrThreads * kScrPer;  // elements per block

template <typename V>
__global__ void __launch_bounds__(kScrThreads) screen_count(const V *__restrict__ f, int64_t K,
                                                            V t, int32_t *__restrict__ cnt) {
    __shared__ int s[kScrThreads / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScrChunk + threadIdx.x * kScrPer;
    int c = 0;
#pragma unroll
    for (int e = 0; e < kScrPer; ++e) c += (base + e < K && f[base + e] > t) ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int total = 0;
        for (int w = 0; w < kScrThreads / 32; ++w) total += s[w];
        cnt[blockIdx.x] = total;
    }
}

template <typename V>
__global__ void __launch_bounds__(kScrThreads) screen_write(const V *__restrict__ f, int64_t K,
                                                            V t,
                                                            const int32_t *__restrict__ cnt,
                                                            int32_t *__restrict__ surv,
                                                            int64_t *__restrict__ m_out) {
    __shared__ int s_warp[kScrThreads / 32];
    __shared__ int64_t s_off;
    if (threadIdx.x == 0) {
        int64_t off = 0;
        for (unsigned b = 0; b < blockIdx.x; ++b) off += cnt[b];
        s_off = off;
        if (blockIdx.x == gridDim.x - 1) *m_out = off + cnt[blockIdx.x];
    }
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScrChunk + threadIdx.x * kScrPer;
    bool pass[kScrPer];
    int c = 0;
#pragma unroll
    for (int e = 0; e < kScrPer; ++e) {
        pass[e] = base + e < K && f[base + e] > t;
        c += pass[e] ? 1 : 0;
    }
    // block-exclusive scan of c in thread order
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int warp_off = 0;
    for (int w = 0; w < warp; ++w) warp_off += s_warp[w];
    int64_t pos = s_off + warp_off + incl - c;
#pragma unroll
    for (int e = 0; e < kScrPer; ++e)
        if (pass[e]) surv[pos++] = static_cast<int32_t>(base + e);
}

}  // namespace

cudaError_t launch_screen(Ctx &c, int64_t k, int64_t t_floor, int64_t *m_dev) {
    if (k <= 0) return cudaMemsetAsync(m_dev, 0, sizeof(int64_t), c.stream);
    const unsigned blocks = static_cast<unsigned>((k + kScrChunk - 1) / kScrChunk);
    screen_count<int64_t><<<blocks, kScrThreads, 0, c.stream>>>(c.f, k, t_floor, c.blk_count);
    screen_write<int64_t><<<blocks, kScrThreads, 0, c.stream>>>(c.f, k, t_floor, c.blk_count, c.surv, m_dev);
    c.launches += 2;
    return cudaSuccess;
}

// real-valued f (a4'): survivors f_k > T compared in binary64
cudaError_t launch_screen_real(Ctx &c, int64_t k, double T, int64_t *m_dev) {
    if (k <= 0) return cudaMemsetAsync(m_dev, 0, sizeof(int64_t), c.stream);
    const unsigned blocks = static_cast<unsigned>((k + kScrChunk - 1) / kScrChunk);
    screen_count<double><<<blocks, kScrThreads, 0, c.stream>>>(c.freal, k, T, c.blk_count);
    screen_write<double><<<blocks, kScrThreads, 0, c.stream>>>(c.freal, k, T, c.blk_count, c.surv, m_dev);
    c.launches += 2;
    return cudaSuccess;
}

}  // namespace ubqp
