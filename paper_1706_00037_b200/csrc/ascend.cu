// ascend.cu — K-ASC: batched steepest ascent on 1-bit flips.
//
// PerformSteepestAscent ("terminating when no improvements are possible or
// a maximum number of flips have been made. No checks for cycling nor tabu lists"), with
// the 1-flip method of Glover et al. 2002:
//     k* = argmax_j Delta_j (lowest j on ties); stop if Delta_k* <= 0 or flips == max;
//     f += Delta_k*;  d = 1 - 2 x_k*;  x_k* ^= 1;
//     Delta_j += 2 d (1 - 2 x_j) Q_{j k*}  (j != k*);   Delta_k* = -Delta_k*.
//
// One CTA per survivor.  The gain vector lives in registers: thread t owns the 4
// consecutive variables j = c*4*BLOCK + 4t + e (e < 4) of every chunk c < NCH, so each
// step streams row k* of Q8 (= column k* by symmetry, n bytes, coalesced 4 B per thread)
// exactly once.  The argmax is a warp __reduce_max/__reduce_min pair plus one
// __syncthreads over double-buffered shared slots; x_k* travels with the winning index.
#include <climits>

#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

template <int BLOCK, int NCH>
__global__ void __launch_bounds__(BLOCK)
ascend_kernel(const int32_t *__restrict__ slots, int64_t m, int max_flips, int n, int n_pad,
              int W64, int64_t k_local, int rank, int world, const int8_t *__restrict__ Q8,
              const int32_t *__restrict__ gains, const int64_t *__restrict__ f_in,
              const uint64_t *__restrict__ Xb, int64_t *__restrict__ f_out,
              int32_t *__restrict__ flips_out, uint64_t *__restrict__ bits_out,
              long long *__restrict__ best_key) {
    constexpr int NW = BLOCK / 32;
    constexpr int CH = 4 * BLOCK;   // variables per chunk
    __shared__ int s_val[2][NW];
    __shared__ unsigned s_idx[2][NW];
    __shared__ uint32_t s_bits[(CH * NCH) / 32];

    const int i = blockIdx.x;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int64_t s = slots[i];
    if (s < 0 || s >= k_local) {               // invalid slot: reported as flips = -1
        if (t == 0) {
            if (flips_out) flips_out[i] = -1;
            if (f_out) f_out[i] = 0;
        }
        return;
    }

    int32_t D[NCH][4];
    uint32_t xm = 0;                            // bit (4c + e) = x_j
    const int32_t *grow = gains + s * n_pad;
    const uint64_t *xrow = Xb + s * W64;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int j0 = c * CH + 4 * t;
        if (j0 < n_pad) {
            const int4 v = *reinterpret_cast<const int4 *>(grow + j0);
            D[c][0] = v.x; D[c][1] = v.y; D[c][2] = v.z; D[c][3] = v.w;
        } else {
            D[c][0] = D[c][1] = D[c][2] = D[c][3] = INT_MIN;
        }
        uint32_t b4 = 0;
        if (j0 < n) b4 = static_cast<uint32_t>(xrow[j0 >> 6] >> (j0 & 63)) & 15u;
        xm |= b4 << (4 * c);
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (j0 + e >= n) D[c][e] = INT_MIN;    // padding is never a candidate
    }
    int64_t fv = f_in[s];
    int flips = 0;
    int par = 0;

    for (;;) {
        // ---- argmax with lowest-index tie-break; carry x_k* in bit 0 of the index key
        int bv = INT_MIN;
        unsigned bk = 0xFFFFFFFFu;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (D[c][e] > bv) {                // strict: first (lowest) j wins ties
                    bv = D[c][e];
                    bk = (static_cast<unsigned>(c * CH + 4 * t + e) << 1) | ((xm >> (4 * c + e)) & 1u);
                }
        const int wv = __reduce_max_sync(0xFFFFFFFFu, bv);
        const unsigned wk = __reduce_min_sync(0xFFFFFFFFu, bv == wv ? bk : 0xFFFFFFFFu);
        if (lane == 0) {
            s_val[par][warp] = wv;
            s_idx[par][warp] = wk;
        }
        __syncthreads();
        int gv = s_val[par][0];
        unsigned gk = s_idx[par][0];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
            const int v = s_val[par][w];
            const unsigned k = s_idx[par][w];
            if (v > gv || (v == gv && k < gk)) { gv = v; gk = k; }
        }
        par ^= 1;
        if (gv <= 0 || flips == max_flips) break;

        // ---- apply the flip of k*
        const int kstar = static_cast<int>(gk >> 1);
        const int d2 = (gk & 1u) ? -2 : 2;         // 2 d, d = 1 - 2 x_k*
        fv += gv;
        ++flips;
        const int8_t *qrow = Q8 + static_cast<int64_t>(kstar) * n_pad;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int j0 = c * CH + 4 * t;
            if (j0 < n_pad) {
                const char4 q = *reinterpret_cast<const char4 *>(qrow + j0);
                const int qq[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int xb = (xm >> (4 * c + e)) & 1;
                    const int coef = xb ? -d2 : d2;  // 2 d (1 - 2 x_j)
                    if (j0 + e == kstar) {
                        D[c][e] = -D[c][e];
                        xm ^= 1u << (4 * c + e);
                    } else {
                        D[c][e] += coef * qq[e];
                    }
                }
            }
        }
    }

    // ---- outputs
    if (bits_out) {
        for (int w = t; w < (CH * NCH) / 32; w += BLOCK) s_bits[w] = 0;
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int j0 = c * CH + 4 * t;
            const uint32_t b4 = (xm >> (4 * c)) & 15u;
            if (b4) atomicOr(&s_bits[j0 >> 5], b4 << (j0 & 31));
        }
        __syncthreads();
        for (int w = t; w < W64; w += BLOCK)
            bits_out[static_cast<int64_t>(i) * W64 + w] =
                static_cast<uint64_t>(s_bits[2 * w]) | (static_cast<uint64_t>(s_bits[2 * w + 1]) << 32);
    }
    if (t == 0) {
        if (f_out) f_out[i] = fv;
        if (flips_out) flips_out[i] = flips;
        if (best_key) {
            const int64_t g = static_cast<int64_t>(rank) + s * world;
            const long long key = static_cast<long long>(
                (static_cast<uint64_t>(fv + (1ll << 40)) << 22) |
                static_cast<uint64_t>((1ll << 22) - 1 - g));
            atomicMax(best_key, key);
        }
    }
}

template <int BLOCK, int NCH>
void launch_inst(Ctx &c, const int32_t *slots, int64_t m, int32_t max_flips, int64_t *f_dev,
                 int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev) {
    ascend_kernel<BLOCK, NCH><<<static_cast<unsigned>(m), BLOCK, 0, c.stream>>>(
        slots, m, max_flips, c.n, c.n_pad, c.W64, c.k_local, c.rank, c.world, c.Q8, c.gains, c.f,
        c.Xb, f_dev, flips_dev, bits_dev, reinterpret_cast<long long *>(best_dev));
}

}  // namespace

// returns 0 on success, 1 if n is outside the instantiated range
int launch_ascend(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                  int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev) {
    if (m <= 0) return 0;
    const int np = c.n_pad;
#define UBQP_ASC(B, N)                                                                 \
    do {                                                                               \
        launch_inst<B, N>(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev); \
        ++c.launches;                                                                  \
        return 0;                                                                      \
    } while (0)
    if (np <= 1024) UBQP_ASC(256, 1);
    if (np <= 2048) UBQP_ASC(256, 2);
    if (np <= 3072) UBQP_ASC(256, 3);
    if (np <= 4096) UBQP_ASC(256, 4);
    if (np <= 5120) UBQP_ASC(256, 5);
    if (np <= 6144) UBQP_ASC(256, 6);
    if (np <= 7168) UBQP_ASC(256, 7);
    if (np <= 8192) UBQP_ASC(256, 8);
    if (np <= 10240) UBQP_ASC(512, 5);
    if (np <= 12288) UBQP_ASC(512, 6);
    if (np <= 14336) UBQP_ASC(512, 7);
    if (np <= 16384) UBQP_ASC(512, 8);
#undef UBQP_ASC
    return 1;
}

}  // namespace ubqp
