// gen.cu — K-GEN: on-device generation of the solution batch.
//
// One thread per (slot, 64-bit word) of the padded row: it produces the packed word
// Xb[slot][w] (w < W64) and its byte expansion X8[slot][64w .. 64w+63] (the int8
// A operand of the evaluation GEMM, zero beyond n).  HBM-write bound:
// n/8 + n_pad bytes per solution.
//
//   Glover diversification (include/ubqp.h ubqp_diversify)
//   SplitMix64 random starts (include/ubqp.h ubqp_random)
#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

// bits -> bytes: 4 bits of `nib` to 4 bytes (LSB first).  nib * (1 + 2^7 + 2^14 + 2^21)
// places bit j at bit 8j with no two partial products overlapping, so no carries.
__device__ __forceinline__ uint32_t spread4(uint32_t nib) {
    return (nib * 0x00204081u) & 0x01010101u;
}

__device__ __forceinline__ void store_expanded(int8_t *dst, uint64_t word) {
    uint32_t o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = spread4(static_cast<uint32_t>(word >> (4 * i)) & 15u);
    int4 *d = reinterpret_cast<int4 *>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i)
        d[i] = make_int4(static_cast<int>(o[4 * i]), static_cast<int>(o[4 * i + 1]),
                         static_cast<int>(o[4 * i + 2]), static_cast<int>(o[4 * i + 3]));
}

__device__ __forceinline__ uint64_t tail_mask(int n, int w) {
    const int rem = n - 64 * w;
    return rem >= 64 ? ~0ull : (rem <= 0 ? 0ull : ((1ull << rem) - 1ull));
}

// floor(sqrt(v)) for 0 <= v < 2^53, exact after correction
__device__ __forceinline__ int64_t isqrt_dev(int64_t v) {
    int64_t s = static_cast<int64_t>(sqrt(static_cast<double>(v)));
    while (s * s > v) --s;
    while ((s + 1) * (s + 1) <= v) ++s;
    return s;
}

// parents == nullptr: Glover (O4), x = seed xor M(h,q), complemented within n iff c = 1.
// parents != nullptr: blend (O4b, R11b), x takes parent[g mod P]'s bits on the mask (its
// complement when c = 1) and the seed's elsewhere: x = seed xor (mask_c & (p xor seed)).
// p = NOT seed gives back the Glover word: seed xor mask_c = seed xor M, complemented iff c.
__global__ void __launch_bounds__(256) glover_kernel(const uint64_t *__restrict__ seed,
                                                     const uint64_t *__restrict__ parents,
                                                     int64_t n_parents, int64_t t0,
                                                     int64_t k, int rank, int world, int B, int n,
                                                     int W64, int NW, int n_pad,
                                                     uint64_t *__restrict__ Xb,
                                                     int8_t *__restrict__ X8) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * NW) return;
    const int64_t slot = idx / NW;
    const int w = static_cast<int>(idx - slot * NW);
    uint64_t word = 0;
    if (w < W64) {
        const int64_t g = global_index(slot, rank, world, B);
        const int64_t period = static_cast<int64_t>(n) * (n + 1);
        int64_t t = (t0 + g) % period;
        if (t < 0) t += period;
        const int64_t h = (1 + isqrt_dev(1 + 4 * t)) / 2;
        const int64_t r = t - h * (h - 1);
        const int64_t q1 = r / 2;              // q - 1
        const bool comp = (r & 1) != 0;
        // M(h,q) restricted to [64w, 64w+64): j = q1 + m h
        const int64_t lo = 64ll * w;
        int64_t j = q1;
        if (j < lo) j = q1 + ((lo - q1 + h - 1) / h) * h;
        uint64_t mask = 0;
        const int64_t hi = lo + 64 < n ? lo + 64 : n;
        for (; j < hi; j += h) mask |= 1ull << (j - lo);
        const uint64_t sw = seed[w];
        const uint64_t diff = parents ? parents[(g % n_parents) * W64 + w] ^ sw : ~0ull;
        word = (sw ^ ((comp ? ~mask : mask) & diff)) & tail_mask(n, w);
        Xb[slot * W64 + w] = word;
    }
    store_expanded(X8 + slot * n_pad + 64ll * w, word);
}

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void __launch_bounds__(256) random_kernel(uint64_t seed, int64_t k, int rank, int world, int B,
                                                     int n, int W64, int NW, int n_pad,
                                                     uint64_t *__restrict__ Xb,
                                                     int8_t *__restrict__ X8) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * NW) return;
    const int64_t slot = idx / NW;
    const int w = static_cast<int>(idx - slot * NW);
    uint64_t word = 0;
    if (w < W64) {
        const uint64_t g = static_cast<uint64_t>(global_index(slot, rank, world, B));
        const uint64_t ctr = g * static_cast<uint64_t>(W64) + static_cast<uint64_t>(w) + 1ull;
        word = splitmix_mix(seed + ctr * 0x9E3779B97F4A7C15ull) & tail_mask(n, w);
        Xb[slot * W64 + w] = word;
    }
    store_expanded(X8 + slot * n_pad + 64ll * w, word);
}

__global__ void __launch_bounds__(256) expand_kernel(int64_t k, int n, int W64, int NW, int n_pad,
                                                     uint64_t *__restrict__ Xb,
                                                     int8_t *__restrict__ X8) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * NW) return;
    const int64_t slot = idx / NW;
    const int w = static_cast<int>(idx - slot * NW);
    uint64_t word = 0;
    if (w < W64) {
        word = Xb[slot * W64 + w] & tail_mask(n, w);
        Xb[slot * W64 + w] = word;
    }
    store_expanded(X8 + slot * n_pad + 64ll * w, word);
}

// bits -> bytes of arbitrary device rows (the re-evaluation of ascended real-Q solutions)
__global__ void __launch_bounds__(256) expand_to_kernel(const uint64_t *__restrict__ bits, int64_t k, int n, int W64,
                                                        int NW, int n_pad, int8_t *__restrict__ X8) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * NW) return;
    const int64_t slot = idx / NW;
    const int w = static_cast<int>(idx - slot * NW);
    const uint64_t word = w < W64 ? bits[slot * W64 + w] & tail_mask(n, w) : 0ull;
    store_expanded(X8 + slot * n_pad + 64ll * w, word);
}

// x_i = [sum_j Q_ij > 0].  One block per 32-bit output word (rows 32w .. 32w+31), each
// of its 8 warps sums 4 rows with 16-byte loads; per plane the row sum fits int32 (n * 127),
// the planes combine exactly in int128 (a real Q's evaluation image, R22: sum_s 128^s rowsum_s).
struct Planes {
    const int8_t *p[kMaxPlanes];
    int count;
};

__global__ void __launch_bounds__(256) first_derivative_kernel(Planes planes, int n, int q_ld,
                                                               uint32_t *__restrict__ bits32) {
    __shared__ uint32_t s_word;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_word = 0;
    __syncthreads();
    for (int r = warp; r < 32; r += 8) {
        const int i = blockIdx.x * 32 + r;
        if (i >= n) break;
        __int128 tot = 0;
        for (int pl = planes.count - 1; pl >= 0; --pl) {
            const int8_t *row = planes.p[pl] + static_cast<int64_t>(i) * q_ld;
            int s = 0;
            for (int j0 = 16 * lane; j0 < n; j0 += 16 * 32) {   // rows are zero padded past n
                const int4 v = *reinterpret_cast<const int4 *>(row + j0);
                const int w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) s = __dp4a(w[q], 0x01010101, s);
            }
            s = __reduce_add_sync(0xffffffffu, s);
            tot = tot * 128 + s;
        }
        if (lane == 0 && tot > 0) atomicOr(&s_word, 1u << r);
    }
    __syncthreads();
    if (threadIdx.x == 0) bits32[blockIdx.x] = s_word;
}

inline unsigned blocks_for(int64_t threads) { return static_cast<unsigned>((threads + 255) / 256); }

}  // namespace

void launch_glover(Ctx &c, const uint64_t *seed_dev, int64_t t0, int64_t k, const uint64_t *parents_dev,
                   int64_t n_parents) {
    if (k <= 0) return;
    const int NW = c.n_pad / 64;
    glover_kernel<<<blocks_for(k * NW), 256, 0, c.stream>>>(seed_dev, parents_dev, n_parents, t0, k, c.rank,
                                                            c.world, c.shard_b, c.n,
                                                            c.W64, NW, c.n_pad, c.Xb, c.X8);
    ++c.launches;
}

void launch_random(Ctx &c, uint64_t seed, int64_t k) {
    if (k <= 0) return;
    const int NW = c.n_pad / 64;
    random_kernel<<<blocks_for(k * NW), 256, 0, c.stream>>>(seed, k, c.rank, c.world, c.shard_b, c.n, c.W64,
                                                            NW, c.n_pad, c.Xb, c.X8);
    ++c.launches;
}

void launch_expand(Ctx &c, int64_t k) {
    if (k <= 0) return;
    const int NW = c.n_pad / 64;
    expand_kernel<<<blocks_for(k * NW), 256, 0, c.stream>>>(k, c.n, c.W64, NW, c.n_pad, c.Xb, c.X8);
    ++c.launches;
}

void launch_first_derivative(Ctx &c, uint64_t *bits_dev) {
    Planes pl{};
    if (c.real) {
        for (int s = 0; s < c.w_limbs; ++s) pl.p[s] = c.Qw[s];
        pl.count = c.w_limbs;
    } else {
        pl.p[0] = c.Q8;
        pl.count = 1;
    }
    // one block per 32-bit word of the W64 output words (2 W64 words, the last may be padding)
    first_derivative_kernel<<<2 * c.W64, 256, 0, c.stream>>>(pl, c.n, c.q_ld, reinterpret_cast<uint32_t *>(bits_dev));
    ++c.launches;
}

void launch_expand_to(Ctx &c, const uint64_t *bits, int64_t k, int8_t *X8dst) {
    if (k <= 0) return;
    const int NW = c.n_pad / 64;
    expand_to_kernel<<<blocks_for(k * NW), 256, 0, c.stream>>>(bits, k, c.n, c.W64, NW, c.n_pad, X8dst);
    ++c.launches;
}

}  // namespace ubqp
