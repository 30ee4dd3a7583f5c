// ascend_warp.cu — K-ASC with ONE WARP per solution.
//
// Same walk as ascend.cu (the 1-flip method of Glover et al. 2002):
//     k* = argmax_j Delta_j (lowest j on ties); stop if Delta_k* <= 0 or flips == max;
//     f += Delta_k*;  d = 1 - 2 x_k*;  x_k* ^= 1;
//     Delta_j += 2 d (1 - 2 x_j) Q_{j k*}  (j != k*);   Delta_k* = -Delta_k*.
//
// Why a second dense kernel: the CTA-of-two-warps kernel (ascend.cu) exchanges its argmax through
// shared memory and bar.sync every step and holds x as byte masks.  Here ONE warp owns all n gains
// of a solution, so the argmax is one warp REDUX + one shuffle, and x lives in the key's sign.
//
// Gains are held as SIGN-FOLDED keys: with key'_j = 256 (Delta_j + 2^21) + (255 - li)
// (li = 16c + e, the lane-local index; key' > 0 since |Delta| <= 254 n - 127 < 2^21),
//     K_j = +key'_j if x_j = 0,   K_j = -key'_j if x_j = 1,
// so the update is UNIFORM over j: K_j += 512 s_k* Q_{k* j} (s = 1 - 2x), one IDP.2A per variable
// that also extracts the byte (dp2a with (C, 0) / (0, C)), and the best key' of a lane is
// max(max_j K_j, -min_j K_j): one 3-input max and one 3-input min per two variables.  Lane L
// owns j = 512c + 16L + e (c < NCH, e < 16), so row k* is staged by coalesced 16-byte cp.async
// copies of each lane's OWN pieces (no cross-lane wait, an L2 round trip; a single bulk copy
// (TMA) measured 1000-1300 cycles of latency per 7 KB row, tools/l2bw.cu) and read back by one
// conflict-free LDS.128 per 16 variables.  The owner of k* fixes its key through one uniform
// jump table (in-place adds, overlapping the copy) and zeroes the staged Q_k*k* byte, so the
// uniform update leaves the new key alone.  Padding variables (j >= n) hold K = 0.
//
// Register budget: 16 NCH keys + ~30 per lane (no spills up to NCH = 14, n_pad <= 7168, at
// 255 registers = 2 warps per SMSP).  Automatic selection uses it for n_pad in (3584, 7168] and
// the 4- and 6-chunk shapes, where it measured faster than the CTA kernel;
// larger n use the multi-warp kernel (ascend_mw.cu, §7.4m).
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ubqp_internal.cuh"
#include "warp_keys.cuh"

namespace ubqp {
namespace {

using namespace dev;

constexpr int kOffW = 1 << 21;

#ifndef UBQP_WARP_SHORT
#define UBQP_WARP_SHORT 1
#endif
template <int NCH, int MINB>
__global__ void __launch_bounds__(32, MINB)
ascend_warp_kernel(const int32_t *__restrict__ slots, int max_flips, int n, int n_pad, int q_ld, int W64,
                   int64_t k_local, int rank, int world, int shard_b, const int8_t *__restrict__ Q8,
                   const int32_t *__restrict__ gains, const int64_t *__restrict__ f_in,
                   const uint64_t *__restrict__ Xb, int64_t *__restrict__ f_out, int32_t *__restrict__ flips_out,
                   uint64_t *__restrict__ bits_out, long long *__restrict__ best_key, int zero) {
    extern __shared__ __align__(128) uint8_t smem[];    // row k* (NCH x 512 bytes)

    const int lane = threadIdx.x;
    const int i = blockIdx.x;
    const int64_t s = slots[i];
    if (s < 0 || s >= k_local) {                   // invalid slot: reported as flips = -1
        if (lane == 0) {
            if (flips_out) flips_out[i] = -1;
            if (f_out) f_out[i] = 0;
        }
        return;
    }

    int K[NCH][16];
    const int32_t *grow = gains + s * n_pad;
    const uint64_t *xrow = Xb + s * W64;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int j0 = 512 * c + 16 * lane;
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
                const int kp = (gg[b] + kOffW) * 256 + (255 - (16 * c + e));
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

    const uint32_t sbuf = smem_u32(smem) + 16 * lane;   // this lane's staged pieces
    const int8_t *qlane = Q8 + 16 * lane;
    int64_t fv = f_in[s];
    int flips = 0;
    int cm0 = mx, cm1 = mx, cn0 = mn, cn1 = mn;    // NCH = 14: chain values carried between steps
    for (;;) {
        // ---- argmax.  Lane best: key' = max(max K, -min K) = (largest Delta, then lowest
        // li = 16c + e).  j = 512c + 16 lane + e orders ties by (c, lane, e), so ONE REDUX over
        // (Delta + OFF) << 9 | (15 - c) << 5 | (31 - lane) (< 2^31) finds the largest Delta, then the
        // lowest j up to e; the winner lane's e and x come by one shuffle.
        const int best = max(mx, -mn);
#if UBQP_WARP_SHORT
        // (Delta + OFF) << 9 | (15 - c) << 5 == (key' >> 4) << 5, since the low byte of key' is
        // 255 - li = (15 - c) << 4 | (15 - e): one shift and one OR before the REDUX; the chunk
        // and lane parts of k* come from the REDUX value while the shuffle is in flight
        const unsigned v = (static_cast<unsigned>(best) >> 4 << 5) | static_cast<unsigned>(31 - lane);
        const unsigned wv = __reduce_max_sync(0xFFFFFFFFu, v);
        const int wl = 31 - static_cast<int>(wv & 31u);
        const int gv = static_cast<int>(wv >> 9) - kOffW;
        const int kbase = 512 * (15 - static_cast<int>((wv >> 5) & 15u)) + 16 * wl;
        const int info = __shfl_sync(0xFFFFFFFFu, (best & 255) | (best != mx ? 256 : 0), wl);
        if (gv <= 0 || flips == max_flips) break;

        // ---- stage row k* (= column k*, Q symmetric): each lane copies its own pieces
        const int li = 255 - (info & 255);
        const int xk = info >> 8;
        const int kstar = kbase + 15 - (info & 15);
        UBQP_DCHECK(kstar == (li >> 4) * 512 + 16 * wl + (li & 15));
#else
        const int lbest = 255 - (best & 255);      // this lane's li
        const unsigned v = (static_cast<unsigned>(best >> 8) << 9) |
                           (static_cast<unsigned>(15 - (lbest >> 4)) << 5) | static_cast<unsigned>(31 - lane);
        const unsigned wv = __reduce_max_sync(0xFFFFFFFFu, v);
        const int wl = 31 - static_cast<int>(wv & 31u);
        const int gv = static_cast<int>(wv >> 9) - kOffW;
        const int info = __shfl_sync(0xFFFFFFFFu, (best & 255) | (best != mx ? 256 : 0), wl);
        if (gv <= 0 || flips == max_flips) break;

        // ---- stage row k* (= column k*, Q symmetric): each lane copies its own pieces
        const int li = 255 - (info & 255);
        const int xk = info >> 8;
        const int kstar = (li >> 4) * 512 + 16 * wl + (li & 15);
#endif
        // 32-bit row offset (kstar * q_ld < 7168 * 7168): a short dependent chain to the copies
        // (measured 1.113 -> 1.169 Gsteps/s at n = 7000 against the 64-bit product)
        UBQP_DCHECK(kstar >= 0 && kstar < n && li < 16 * NCH && 512 * NCH <= q_ld);
        const int8_t *src = qlane + static_cast<uint32_t>(kstar) * static_cast<uint32_t>(q_ld);
#pragma unroll
        for (int c = 0; c < NCH; ++c) cp_async16(sbuf + 512 * c, src + 512 * c);
        cp_async_commit();
        fv += gv;
        ++flips;
        // ---- owner of k*: x flips and Delta -> -Delta, i.e. K_new = -s (256 (OFF - Delta) + 255 - li);
        // the row byte Q_k*k* is zeroed below so the uniform update leaves the new key alone
        const int C = xk ? -512 : 512;             // 512 s_k*
        const bool owner = lane == wl;
        {
            const int kp = (kOffW - gv) * 256 + (255 - li);
            const int corr = owner ? (xk ? kp : -kp) - (xk ? -best : best) : 0;
            add_key<NCH>(K, li, corr);
        }
        cp_async_wait();                           // this lane's own pieces only
        UBQP_DCHECK(!owner || (li >> 4) < NCH);
        if (owner) asm volatile("st.shared.u8 [%0], %1;" ::"r"(sbuf + 512 * (li >> 4) + (li & 15)), "r"(0) : "memory");

        // ---- fused uniform update + next argmax (max chains and min chains over K)
        const uint32_t a0 = static_cast<uint32_t>(C) & 0xFFFFu;   // (C, 0): picks bytes 0 / 2
        const uint32_t a1 = static_cast<uint32_t>(C) << 16;       // (0, C): picks bytes 1 / 3
        // The chains restart from INT_MIN / INT_MAX every step.  At NCH = 14 they restart through
        // their previous values and the run-time zero `zero` (a loop-carried dependency ptxas
        // cannot see through), which changes ptxas's schedule of the step: measured same-box
        // n = 7000 1.113 vs 1.086 Gsteps/s; at n = 5000 the same form measured 1.45 vs 1.51, so
        // the other shapes keep constant starts.
        int m0 = INT_MIN, m1 = INT_MIN, n0 = INT_MAX, n1 = INT_MAX;
        if constexpr (NCH == 14) {
            m0 = INT_MIN | (cm0 & zero);
            m1 = INT_MIN | (cm1 & zero);
            n0 = INT_MAX & ~(cn0 & zero);
            n1 = INT_MAX & ~(cn1 & zero);
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const uint32_t addr = sbuf + 512 * c;
            uint4 w;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(addr)
                         : "memory");
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
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
        if constexpr (NCH == 14) {
            cm0 = m0;
            cm1 = m1;
            cn0 = n0;
            cn1 = n1;
        }
    }

    // ---- outputs: x_j = [K_j < 0], 16 bits per chunk at j0 = 512 c + 16 lane (16-bit aligned)
    if (bits_out) {
        uint16_t *bo = reinterpret_cast<uint16_t *>(bits_out + static_cast<int64_t>(i) * W64);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            uint32_t b16 = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) b16 |= (K[c][e] < 0 ? 1u : 0u) << e;
            const int w16 = 32 * c + lane;
            if (w16 < 4 * W64) bo[w16] = static_cast<uint16_t>(b16);
        }
    }
    if (lane == 0) {
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

template <int NCH>
void launch_w(Ctx &c, const int32_t *slots, int64_t m, int32_t max_flips, int64_t *f_dev, int32_t *flips_dev,
              uint64_t *bits_dev, int64_t *best_dev) {
    // registers ~ 16 NCH keys + ~32; the register file is split per SMSP (16 K each), so the
    // resident warps per SM are 4 x floor(512 / registers): 8 at NCH = 14 (<= 255 registers)
    // NCH = 9 fits 166 registers (3 warps per SMSP instead of 2): measured n = 4500 1.753 vs
    // 1.563 Gsteps/s (profiles/r02_warp_slack.log); a 16-register slack elsewhere gained nothing
    // (n = 2500: 2.79 vs 2.96 at 5 warps per SMSP) and spills at NCH = 3
#ifndef UBQP_WARP_REGS_SLACK
#define UBQP_WARP_REGS_SLACK 32   // A/B: the non-key registers budgeted per lane
#endif
    constexpr int kSlack = NCH == 9 ? 22 : UBQP_WARP_REGS_SLACK;
    constexpr int kRegsB = ((16 * NCH + kSlack + 7) / 8) * 8;
    constexpr int kMinB = 4 * (512 / kRegsB) > 32 ? 32 : 4 * (512 / kRegsB);
    static const size_t smem_extra = [] {     // occupancy experiments: pad the CTA's shared memory
        const char *e = getenv("UBQP_ASC_WARP_SMEM");
        return static_cast<size_t>(e ? atoi(e) : 0);
    }();
    const size_t smem = 512 * NCH + smem_extra;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(ascend_warp_kernel<NCH, kMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    ascend_warp_kernel<NCH, kMinB><<<static_cast<unsigned>(m), 32, smem, c.stream>>>(
        slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
        c.Xb, f_dev, flips_dev, bits_dev, reinterpret_cast<long long *>(best_dev), 0);
}

}  // namespace

int ascend_warp_max_n() { return 14 * 512; }

int launch_ascend_warp(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                       int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev) {
    if (m <= 0) return 0;
    const int nch = (c.n_pad + 511) / 512;
    if (nch > 14 || nch * 512 > c.q_ld) return 1;
    switch (nch) {
#define UBQP_WCASE(N) \
    case N: launch_w<N>(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev); break;
        UBQP_WCASE(1) UBQP_WCASE(2) UBQP_WCASE(3) UBQP_WCASE(4) UBQP_WCASE(5) UBQP_WCASE(6) UBQP_WCASE(7)
        UBQP_WCASE(8) UBQP_WCASE(9) UBQP_WCASE(10) UBQP_WCASE(11) UBQP_WCASE(12) UBQP_WCASE(13) UBQP_WCASE(14)
#undef UBQP_WCASE
        default: return 1;
    }
    ++c.launches;
    return 0;
}

}  // namespace ubqp
