// ascend_mw.cu — K-ASC with 2-4 WARPS per solution (n_pad > 7168).
//
// The walk of ascend.cu / ascend_warp.cu: k* = argmax_j Delta_j (lowest j on
// ties), stop if Delta_k* <= 0 or flips == max, f += Delta_k*, x_k* ^= 1, Delta_j += 2 d (1 - 2x_j)
// Q_jk* (j != k*), Delta_k* = -Delta_k*.  Same sign-folded keys and uniform dp2a update as the
// one-warp kernel (ascend_warp.cu header), spread over NW warps when 16 keys x NCH chunks per
// lane no longer fit one warp's registers.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ubqp_internal.cuh"
#include "warp_keys.cuh"

namespace ubqp {
namespace {

using namespace dev;

constexpr int kOffM = 1 << 22;   // |Delta| <= 254 n - 127 < 2^22 up to n = 16384

// ---- NW warps per solution (n_pad > 7168, and A/B below it; NW in {2, 3, 4}).  Same keys and
// update as the one-warp kernel, with the key offset 2^22 (|Delta| <= 254 n - 127 < 2^22 up to
// n = 16384, and 256 (Delta + 2^22) + 255 < 2^31); warp w of the CTA owns
// j = 512 (NW c + w) + 16 L + e, so the row k* is staged in shared memory in natural order and
// every lane still copies and reads only its own pieces.  The argmax is the warp REDUX + shuffle,
// then ONE cross-warp exchange: each warp's lane 0 publishes a 64-bit word (Delta + OFF, 15 - c,
// NW - 1 - w, 31 - L, key byte, x) into a double-buffered slot (the slot of step t is rewritten
// at t + 2, after every warp passed the barrier of t + 1), one bar.sync, and every warp takes the
// max of the NW words: the largest Delta, then the lowest j = (c, w, L, e).
template <int NCH, int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB)
ascend_mw_kernel(const int32_t *__restrict__ slots, int max_flips, int n, int n_pad, int q_ld, int W64,
                 int64_t k_local, int rank, int world, int shard_b, const int8_t *__restrict__ Q8,
                 const int32_t *__restrict__ gains, const int64_t *__restrict__ f_in,
                 const uint64_t *__restrict__ Xb, int64_t *__restrict__ f_out, int32_t *__restrict__ flips_out,
                 uint64_t *__restrict__ bits_out, long long *__restrict__ best_key) {
    extern __shared__ __align__(128) uint8_t smem[];    // row k* (NW NCH 512 bytes), 2 x 4 exchange words

    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int i = blockIdx.x;
    const int64_t s = slots[i];
    if (s < 0 || s >= k_local) {                   // invalid slot (CTA-uniform): flips = -1
        if (threadIdx.x == 0) {
            if (flips_out) flips_out[i] = -1;
            if (f_out) f_out[i] = 0;
        }
        return;
    }

    int K[NCH][16];
    const int32_t *grow = gains + s * n_pad;
    const uint64_t *xrow = Xb + s * W64;
    const int jl = 512 * w + 16 * lane;            // j of this lane's piece in chunk 0
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int j0 = 512 * NW * c + jl;
        uint32_t bits16 = 0;
        if (j0 < n) bits16 = static_cast<uint32_t>(xrow[j0 >> 6] >> (j0 & 63)) & 0xFFFFu;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            int4 g = make_int4(0, 0, 0, 0);
            if (j0 < n_pad) g = __ldcs(reinterpret_cast<const int4 *>(grow + j0 + 4 * q4));
            const int gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int e = 4 * q4 + b;
                const int kp = (gg[b] + kOffM) * 256 + (255 - (16 * c + e));
                K[c][e] = (j0 + e < n) ? (((bits16 >> e) & 1u) ? -kp : kp) : 0;
            }
        }
    }
    int mx = INT_MIN, mn = INT_MAX;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            mx = max(mx, K[c][e]);
            mn = min(mn, K[c][e]);
        }

    const uint32_t sbuf = smem_u32(smem) + jl;     // this lane's staged pieces (chunk stride 512 NW)
    const uint32_t xw = smem_u32(smem) + 512 * NW * NCH;
    // pieces past the padded row (q_ld) are never copied: zero them once (own pieces, no sync)
    const bool last_ok = 512 * NW * (NCH - 1) + jl < q_ld;
    if (!last_ok)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(sbuf + 512 * NW * (NCH - 1)), "r"(0)
                     : "memory");
    const int8_t *qlane = Q8 + jl;
    int64_t fv = f_in[s];
    int flips = 0;
    uint32_t par = 0;
    for (;;) {
        const int best = max(mx, -mn);
        const unsigned v = (static_cast<unsigned>(best) >> 4 << 5) | static_cast<unsigned>(31 - lane);
        const unsigned wv = __reduce_max_sync(0xFFFFFFFFu, v);
        const int wl = 31 - static_cast<int>(wv & 31u);
        const int info = __shfl_sync(0xFFFFFFFFu, (best & 255) | (best != mx ? 256 : 0), wl);
        if (lane == 0) {
            const uint64_t word = (static_cast<uint64_t>(wv >> 5) << 16) |
                                  (static_cast<uint64_t>(NW - 1 - w) << 14) |
                                  (static_cast<uint64_t>(31 - wl) << 9) | static_cast<uint64_t>(info);
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(xw + 32 * par + 8 * w), "l"(word) : "memory");
        }
        __syncthreads();
        uint64_t W;
        {
            uint64_t a, b;
            asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(xw + 32 * par) : "memory");
            W = a > b ? a : b;
            if constexpr (NW == 3) {
                uint64_t d;
                asm volatile("ld.shared.u64 %0, [%1];" : "=l"(d) : "r"(xw + 32 * par + 16) : "memory");
                W = W > d ? W : d;
            }
            if constexpr (NW == 4) {
                uint64_t d, e;
                asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(d), "=l"(e) : "r"(xw + 32 * par + 16) : "memory");
                d = d > e ? d : e;
                W = W > d ? W : d;
            }
        }
        par ^= 1u;
        const uint32_t hi = static_cast<uint32_t>(W >> 16);              // (Delta + OFF) << 4 | 15 - c
        const int gv = static_cast<int>(hi >> 4) - kOffM;
        if (gv <= 0 || flips == max_flips) break;   // CTA-uniform

        const uint32_t lo = static_cast<uint32_t>(W);
        const int ws = NW - 1 - static_cast<int>((lo >> 14) & 3u);
        const int ls = 31 - static_cast<int>((lo >> 9) & 31u);
        const int li = 255 - static_cast<int>(lo & 255u);
        const int xk = static_cast<int>((lo >> 8) & 1u);
        const int kstar = 512 * (NW * (li >> 4) + ws) + 16 * ls + (li & 15);
        UBQP_DCHECK(15 - static_cast<int>(hi & 15u) == (li >> 4));
        UBQP_DCHECK(kstar >= 0 && kstar < n && li < 16 * NCH && ws < NW);
        const int8_t *src = qlane + static_cast<uint32_t>(kstar) * static_cast<uint32_t>(q_ld);
#pragma unroll
        for (int c = 0; c < NCH; ++c)
            if (c < NCH - 1 || last_ok) cp_async16(sbuf + 512 * NW * c, src + 512 * NW * c);
        cp_async_commit();
        fv += gv;
        ++flips;
        const int C = xk ? -512 : 512;             // 512 s_k*
        const bool owner = w == ws && lane == ls;
        if (w == ws) {                             // warp-uniform: the owner's warp fixes its key
            const int kp = (kOffM - gv) * 256 + (255 - li);
            const int corr = owner ? (xk ? kp : -kp) - (xk ? -best : best) : 0;
            add_key<NCH>(K, li, corr);
        }
        cp_async_wait();
        if (owner)
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(sbuf + 512 * NW * (li >> 4) + (li & 15)), "r"(0) : "memory");

        const uint32_t a0 = static_cast<uint32_t>(C) & 0xFFFFu;
        const uint32_t a1 = static_cast<uint32_t>(C) << 16;
        int m0 = INT_MIN, m1 = INT_MIN, n0 = INT_MAX, n1 = INT_MAX;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const uint32_t addr = sbuf + 512 * NW * c;
            uint4 q;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                         : "r"(addr)
                         : "memory");
            const uint32_t ww[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) {
                int &k0 = K[c][4 * wi + 0];
                int &k1 = K[c][4 * wi + 1];
                int &k2 = K[c][4 * wi + 2];
                int &k3 = K[c][4 * wi + 3];
                k0 = dp2a_lo(a0, ww[wi], k0);
                k1 = dp2a_lo(a1, ww[wi], k1);
                k2 = dp2a_hi(a0, ww[wi], k2);
                k3 = dp2a_hi(a1, ww[wi], k3);
                m0 = max3i(m0, k0, k1);
                n0 = min3i(n0, k0, k1);
                m1 = max3i(m1, k2, k3);
                n1 = min3i(n1, k2, k3);
            }
        }
        mx = max(m0, m1);
        mn = min(n0, n1);
    }

    if (bits_out) {
        uint16_t *bo = reinterpret_cast<uint16_t *>(bits_out + static_cast<int64_t>(i) * W64);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            uint32_t b16 = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) b16 |= (K[c][e] < 0 ? 1u : 0u) << e;
            const int w16 = 32 * (NW * c + w) + lane;
            if (w16 < 4 * W64) bo[w16] = static_cast<uint16_t>(b16);
        }
    }
    if (threadIdx.x == 0) {
        if (f_out) f_out[i] = fv;
        if (flips_out) flips_out[i] = flips;
        if (best_key) {
            const int64_t g = global_index(s, rank, world, shard_b);
            const long long key = static_cast<long long>((static_cast<uint64_t>(fv + (1ll << 40)) << 22) |
                                                         static_cast<uint64_t>((1ll << 22) - 1 - g));
            atomicMax(best_key, key);
        }
    }
}

template <int NCH, int NW>
void launch_mw(Ctx &c, const int32_t *slots, int64_t m, int32_t max_flips, int64_t *f_dev, int32_t *flips_dev,
               uint64_t *bits_dev, int64_t *best_dev) {
    // NCH = 9 fits 168 registers (3 warps per SMSP), as in the one-warp kernel
#ifndef UBQP_MW_SLACK7
#define UBQP_MW_SLACK7 36   // A/B: the non-key register budget at NCH = 7
#endif
#ifndef UBQP_MW_SLACK5
#define UBQP_MW_SLACK5 36   // A/B: the non-key register budget at NCH = 5
#endif
    constexpr int kRegs = ((16 * NCH + (NCH == 9 ? 22 : (NCH == 7 ? UBQP_MW_SLACK7 : (NCH == 5 ? UBQP_MW_SLACK5 : 36))) + 7) / 8) * 8;
    constexpr int kWarps = 4 * (512 / kRegs) > 32 ? 32 : 4 * (512 / kRegs);
    constexpr int kMinB = kWarps / NW < 1 ? 1 : kWarps / NW;
    const size_t smem = 512 * NW * NCH + 64;   // + 2 x 4 exchange words (16-byte aligned pairs)
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(ascend_mw_kernel<NCH, NW, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    ascend_mw_kernel<NCH, NW, kMinB><<<static_cast<unsigned>(m), 32 * NW, smem, c.stream>>>(
        slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
        c.Xb, f_dev, flips_dev, bits_dev, reinterpret_cast<long long *>(best_dev));
}

}  // namespace

// Shapes: NW = 2 (NCH 1..14), 3 (NCH 4..11), 4 (NCH 3..8).  Default: 2 warps up to n_pad = 14336,
// 4 above (NCH = 8: 159 registers, 3 solutions per SM; 3 warps x 11 chunks needs 215 registers,
// 2 solutions per SM).  Measured (tools/asc_micro.py, profiles/r02_mw_micro.log): n = 16000
// 0.335 (NW 4) vs 0.240 (NW 2, 3) Gsteps/s, n = 14336 0.424 (NW 2) vs 0.375 (NW 4).
// UBQP_ASC_MW_NW forces 2, 3 or 4 where that shape is instantiated (A/B).
static bool mw_shape(int nw, int nch) {
    return (nw == 2 && nch >= 1 && nch <= 14) || (nw == 3 && nch >= 4 && nch <= 11) ||
           (nw == 4 && nch >= 3 && nch <= 8);
}
static int mw_warps(int n_pad, int &nch) {
    static const int forced = [] {
        const char *e = getenv("UBQP_ASC_MW_NW");
        return e ? atoi(e) : 0;
    }();
    auto chunks = [n_pad](int nw) { return (n_pad + 512 * nw - 1) / (512 * nw); };
    int nw = chunks(2) <= 14 ? 2 : 4;
    if (forced >= 2 && forced <= 4 && mw_shape(forced, chunks(forced))) nw = forced;
    nch = chunks(nw);
    return nw;
}

int ascend_mw_max_n() { return 16384; }

int launch_ascend_mw(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                     int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev) {
    if (m <= 0) return 0;
    int nch = 0;
    const int nw = mw_warps(c.n_pad, nch);
    if (!mw_shape(nw, nch)) return 1;
#define UBQP_MCASE(W, N) \
    if (nw == W && nch == N) launch_mw<N, W>(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev);
    UBQP_MCASE(2, 1) UBQP_MCASE(2, 2) UBQP_MCASE(2, 3) UBQP_MCASE(2, 4) UBQP_MCASE(2, 5) UBQP_MCASE(2, 6)
    UBQP_MCASE(2, 7) UBQP_MCASE(2, 8) UBQP_MCASE(2, 9) UBQP_MCASE(2, 10) UBQP_MCASE(2, 11) UBQP_MCASE(2, 12)
    UBQP_MCASE(2, 13) UBQP_MCASE(2, 14)
    UBQP_MCASE(3, 4) UBQP_MCASE(3, 5) UBQP_MCASE(3, 6) UBQP_MCASE(3, 7) UBQP_MCASE(3, 8) UBQP_MCASE(3, 9)
    UBQP_MCASE(3, 10) UBQP_MCASE(3, 11)
    UBQP_MCASE(4, 3) UBQP_MCASE(4, 4) UBQP_MCASE(4, 5) UBQP_MCASE(4, 6) UBQP_MCASE(4, 7) UBQP_MCASE(4, 8)
#undef UBQP_MCASE
    ++c.launches;
    return 0;
}

}  // namespace ubqp
