// ascend_real.cu — K-ASC for real-valued Q (reading R20, §7.2′).
//
// PerformSteepestAscent with the 1-flip gains of P:53 on the load-time
// fixed-point image Qt = rint(Q 2^e) (the integer the a4′ limb planes encode), so the walk
// is exact in int64 and f = 2^-e f~:
//     k* = argmax_j Delta_j (lowest j on ties); stop if Delta_k* <= 0 or flips == max_flips;
//     f~ += Delta_k*;  d = 1 - 2 x_k*;  Delta_j += 2 d (1 - 2 x_j) Qt_{j k*};  Delta_k* = -Delta_k*.
// One CTA of 256 threads per survivor; thread t owns j = t + 256 i (i < NPT), gains as
// int64 registers, x as a bit mask; a step streams row k* of Qt (int32, 4 n bytes, HBM:
// Qt does not fit L2 at n = 7000), coalesced 128 B per warp and index.
// The initial int64 gains come from the tensor-core plane evaluations:
//     Delta~ = Qt_jj + sum_s 128^s * 2 (1 - 2 x_j) Y_s,   Y_s = X L_s   (gains_combine_kernel).
#include <climits>
#include <cstdio>

#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

constexpr int kRB = 256;                 // threads per solution
constexpr long long kRPad = LLONG_MIN / 2;   // padding / parked keys: never the maximum

// gains64 (+)= gains << 7 plane (plane 0 starts from the walk diagonal Qt_jj); with the last
// plane, also f~28 = sum_s 128^s f_s of every row (the walk's starting value)
__global__ void __launch_bounds__(256) gains_combine_kernel(const int32_t *__restrict__ g32,
                                                            int64_t *__restrict__ g64,
                                                            const int32_t *__restrict__ diagt, int64_t k,
                                                            int n_pad, int shift, int first,
                                                            const int64_t *__restrict__ fs, int64_t k_max,
                                                            int64_t *__restrict__ fint) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * n_pad) return;
    const int j = static_cast<int>(idx % n_pad);
    const int64_t base = first ? static_cast<int64_t>(diagt[j]) : g64[idx];
    g64[idx] = base + (static_cast<int64_t>(g32[idx]) << shift);
    if (fint && j == 0) {
        const int64_t row = idx / n_pad;
        int64_t v = 0;
        for (int s = kSlices - 1; s >= 0; --s) v = v * 128 + fs[s * k_max + row];
        fint[row] = v;
    }
}

template <int NPT, int MINB>
__global__ void __launch_bounds__(kRB, MINB)
ascend_real_kernel(const int32_t *__restrict__ slots, int max_flips, int n, int n_pad, int qt_ld, int W64,
                   int64_t k_local, const int32_t *__restrict__ Qt, const int64_t *__restrict__ g64,
                   const int64_t *__restrict__ fint_in, const uint64_t *__restrict__ Xb, int q_exp,
                   double *__restrict__ f_out, int64_t *__restrict__ fint_out, int32_t *__restrict__ flips_out,
                   uint64_t *__restrict__ bits_out) {
    constexpr int NW = kRB / 32;
    __shared__ long long s_v[2][NW];
    __shared__ unsigned s_j[2][NW];
    __shared__ uint32_t s_bits[(kRB * NPT) / 32];

    const int i = blockIdx.x;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int64_t s = slots[i];
    if (s < 0 || s >= k_local) {
        if (t == 0) {
            if (flips_out) flips_out[i] = -1;
            if (f_out) f_out[i] = 0.0;
            if (fint_out) fint_out[i] = 0;
        }
        return;
    }
    // gains in shared memory, [q][t] (conflict-free 8-byte words): 3 solutions per SM at
    // n = 7000 instead of 2 with register gains (the step waits on an HBM row fetch, so
    // solutions in flight set the rate)
    extern __shared__ long long s_G[];
    uint64_t xm = 0;
    const int64_t *grow = g64 + s * n_pad;
    const uint64_t *xrow = Xb + s * W64;
    // stored as 64 Delta + (63 - q): one 64-bit max orders (gain, then lowest q)
    long long bk = LLONG_MIN;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        const int j = t + kRB * q;
        const long long g = j < n ? grow[j] * 64 + (63 - q) : kRPad;
        s_G[q * kRB + t] = g;
        bk = max(bk, g);
        if (j < n) xm |= ((xrow[j >> 6] >> (j & 63)) & 1ull) << q;
    }
    long long fv = fint_in[s];
    int flips = 0;
    for (;;) {
        // ---- argmax: thread (tracked by the last update) -> warp (largest gain, then lowest j) -> block
        const int bq = 63 - static_cast<int>(bk & 63);
        long long bv = bk >> 6;
        unsigned bj = (static_cast<unsigned>(t + kRB * bq) << 1) | static_cast<unsigned>((xm >> bq) & 1ull);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const long long ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
            const unsigned oj = __shfl_xor_sync(0xFFFFFFFFu, bj, o);
            if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
        }
        const int par = flips & 1;
        if (lane == 0) {
            s_v[par][warp] = bv;
            s_j[par][warp] = bj;
        }
        __syncthreads();
        long long gv = s_v[par][0];
        unsigned gj = s_j[par][0];
#pragma unroll
        for (int w2 = 1; w2 < NW; ++w2) {
            const long long v = s_v[par][w2];
            const unsigned j2 = s_j[par][w2];
            if (v > gv || (v == gv && j2 < gj)) { gv = v; gj = j2; }
        }
        if (gv <= 0 || flips == max_flips) break;

        // ---- flip k*: update every gain and track the next thread maximum
        const int kstar = static_cast<int>(gj >> 1);
        const long long d2 = (gj & 1u) ? -2 : 2;          // 2 d, d = 1 - 2 x_k*
        fv += gv;
        ++flips;
        const int32_t *row = Qt + static_cast<int64_t>(kstar) * qt_ld + t;
        const int own = (kstar % kRB) == t ? kstar / kRB : -1;
        int32_t qv[NPT];
#pragma unroll
        for (int q = 0; q < NPT; ++q) qv[q] = __ldg(row + kRB * q);   // rows padded to qt_ld
        // the owner parks Delta_k* out of reach of the max for the uniform pass, then stores -gv
        if (own >= 0) s_G[own * kRB + t] = kRPad;
        const int c2 = static_cast<int>(d2) * 64;
        bk = LLONG_MIN;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            const int coef = ((xm >> q) & 1ull) ? -c2 : c2;           // 64 * 2 d (1 - 2 x_j)
            const long long g = s_G[q * kRB + t] + static_cast<long long>(coef) * qv[q];   // IMAD.WIDE
            s_G[q * kRB + t] = g;
            bk = max(bk, g);
        }
        if (own >= 0) {
            const long long g = -gv * 64 + (63 - own);
            s_G[own * kRB + t] = g;
            bk = max(bk, g);
            xm ^= 1ull << own;
        }
    }

    // ---- outputs
    if (bits_out) {
        for (int w2 = t; w2 < (kRB * NPT) / 32; w2 += kRB) s_bits[w2] = 0;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NPT; ++q)
            if ((xm >> q) & 1ull) {
                const int j = t + kRB * q;
                atomicOr(&s_bits[j >> 5], 1u << (j & 31));
            }
        __syncthreads();
        for (int w2 = t; w2 < W64; w2 += kRB)
            bits_out[static_cast<int64_t>(i) * W64 + w2] =
                static_cast<uint64_t>(s_bits[2 * w2]) | (static_cast<uint64_t>(s_bits[2 * w2 + 1]) << 32);
    }
    if (t == 0) {
        if (fint_out) fint_out[i] = fv;
        if (f_out) f_out[i] = ldexp(static_cast<double>(fv), -q_exp);
        if (flips_out) flips_out[i] = flips;
    }
}

template <int NPT>
void launch_real_inst(Ctx &c, const int32_t *slots, int64_t m, int32_t max_flips, double *f_dev, int64_t *fint_dev,
                      int32_t *flips_dev, uint64_t *bits_dev) {
    constexpr int kSmem = NPT * kRB * 8;
    constexpr int kByS = (228 * 1024) / (kSmem + 3 * 1024);
    constexpr int kByR = 65536 / (kRB * (NPT + 40));
    constexpr int kMinB = (kByS < kByR ? kByS : kByR) < 1 ? 1 : (kByS < kByR ? kByS : kByR);
    // > 48 KB dynamic opt-in: per device context, so set before every launch (cheap) rather
    // than once per process (a second device would otherwise fail to launch)
    cudaFuncSetAttribute(ascend_real_kernel<NPT, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    ascend_real_kernel<NPT, kMinB><<<static_cast<unsigned>(m), kRB, kSmem, c.stream>>>(
        slots, max_flips, c.n, c.n_pad, c.qt_ld, c.W64, c.k_local, c.Qt, c.gains64, c.fint, c.Xb, c.q_exp, f_dev,
        fint_dev, flips_dev, bits_dev);
}

}  // namespace

int real_qt_ld(int n_pad) {
    int npt = (n_pad + kRB - 1) / kRB;
    npt = (npt + 3) / 4 * 4;
    return npt * kRB;
}

void launch_gains_combine(Ctx &c, int64_t k, int plane) {
    if (k <= 0) return;
    const int64_t tot = k * c.n_pad;
    gains_combine_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, c.stream>>>(
        c.gains, c.gains64, c.diagt, k, c.n_pad, 7 * plane, plane == 0 ? 1 : 0, c.fs, c.k_max,
        plane == kSlices - 1 ? c.fint : nullptr);
    ++c.launches;
}

int launch_ascend_real(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, double *f_dev,
                       int64_t *fint_dev, int32_t *flips_dev, uint64_t *bits_dev) {
    if (m <= 0) return 0;
    const int npt = c.qt_ld / kRB;
#define UBQP_RI(N)                                                                           \
    if (npt == N) {                                                                          \
        launch_real_inst<N>(c, slots_dev, m, max_flips, f_dev, fint_dev, flips_dev, bits_dev); \
        ++c.launches;                                                                        \
        return 0;                                                                            \
    }
    UBQP_RI(4) UBQP_RI(8) UBQP_RI(12) UBQP_RI(16) UBQP_RI(20) UBQP_RI(24) UBQP_RI(28) UBQP_RI(32)
    UBQP_RI(36) UBQP_RI(40) UBQP_RI(44) UBQP_RI(48) UBQP_RI(52) UBQP_RI(56) UBQP_RI(60) UBQP_RI(64)
#undef UBQP_RI
    return 1;
}

}  // namespace ubqp
