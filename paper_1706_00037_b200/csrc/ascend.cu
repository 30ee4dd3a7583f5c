// ascend.cu — K-ASC: batched steepest ascent on 1-bit flips.
//
// PerformSteepestAscent ("terminating when no improvements are possible or
// a maximum number of flips have been made. No checks for cycling nor tabu lists"), with
// the 1-flip method of Glover et al. 2002:
//     k* = argmax_j Delta_j (lowest j on ties); stop if Delta_k* <= 0 or flips == max;
//     f += Delta_k*;  d = 1 - 2 x_k*;  x_k* ^= 1;
//     Delta_j += 2 d (1 - 2 x_j) Q_{j k*}  (j != k*);   Delta_k* = -Delta_k*.
//
// One CTA of BLOCK threads per survivor; thread t owns the 16 consecutive variables
// j = c*16*BLOCK + 16t + e (e < 16) of every chunk c < NCH, so a step streams row k* of
// Q8 (= column k*, Q symmetric; n bytes) with one 16-byte load per chunk.  Each gain is
// held in a register as a totally ordered key
//     K_j = 256 Delta_j + 2 (127 - li) + x_j          (li = 16c + e, the local index)
// so the running argmax (largest Delta, then lowest j) is a 3-input IMNMX per two
// elements, and the update K_j += C s_j Q_{k* j} (C = 512 d, block-uniform) is one IDP.2A
// per element on FMA pipe: x is held as byte masks m (0xFF where x = 1), t = q ^ m is the
// ones' complement of the negated bytes, and the (t_e, m_e) byte pairs dotted with
// (C, -C) give C (t_e - m_e) = C s_e q_e exactly.  Per 4 elements and step: 1 LOP3 +
// 2 PRMT + 2 IMNMX3 (ALU pipe) and 4 IDP.2A (FMA pipe).  The owner of k* pre-compensates
// K_k* through a two-level jump table (chunk, then element) so the fused loop needs no
// per-element test.  Argmax across lanes: __reduce_max/min_sync; across warps: one
// __syncthreads over double-buffered shared slots holding each warp's winner as one
// orderable 64-bit word.  Codegen sits at the 168-register cap: A/B any edit on one box
// (tools/ab.sh) -- DESIGN.md §13 lists the measured variants.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

constexpr int kPad = -(1 << 30);     // key of padding variables: below every real key

__device__ __forceinline__ int sext_byte(uint32_t w, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "r"(sel));
    return static_cast<int>(r);
}
// selector: byte b in the low byte, its sign replicated above
__device__ __forceinline__ constexpr uint32_t sel_of(int b) {
    return static_cast<uint32_t>(b) | ((8u | b) << 4) | ((8u | b) << 8) | ((8u | b) << 12);
}
// c + a.s16[0] * b.s8[0|2] + a.s16[1] * b.s8[1|3]  (IDP.2A)
__device__ __forceinline__ int dp2a_lo(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t byte_mask_of_nibble(uint32_t nib) {
    return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
}
__device__ __forceinline__ uint32_t nibble_of_byte_mask(uint32_t m) {
    return (((m & 0x01010101u) * 0x01020408u) >> 24) & 0xFu;
}
__device__ __forceinline__ uint32_t word_of(const uint4 &v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

template <int BLOCK, int NCH>
struct Asc {
    static constexpr int E = 16 * NCH;      // variables per thread
    static constexpr int CHUNK = 16 * BLOCK;
    static constexpr int NW = BLOCK / 32;
};

// Owner of k*: pre-set K so that after the uniform update (+C s_new q_kk = -512 q_kk) it
// equals 256(-Delta_old) + 2(127 - li) + x_new, and flip x's byte mask.
template <int L, int NCH>
__device__ __forceinline__ void owner_fix(int (&K)[NCH][16], uint32_t (&m)[NCH][4],
                                          const uint4 (&w)[NCH], int gv, int x_new, int off) {
    constexpr int c = L >> 4, e = L & 15, wi = e >> 2, b = e & 3;
    if constexpr (c < NCH) {
        const int qkk = sext_byte(word_of(w[c], wi), sel_of(b));
        K[c][e] = -gv * 256 + 2 * (127 - L) + x_new + 512 * qkk - off;
        m[c][wi] ^= 0xFFu << (8 * b);
    }
}

template <int C, int NCH>
__device__ __forceinline__ void owner_fix_chunk(int (&K)[NCH][16], uint32_t (&m)[NCH][4],
                                                const uint4 (&w)[NCH], int e, int gv, int x_new, int off) {
#define UBQP_ECASE(E) \
    case E:           \
        owner_fix<C * 16 + E, NCH>(K, m, w, gv, x_new, off); \
        break;
    switch (e) {
        UBQP_ECASE(0) UBQP_ECASE(1) UBQP_ECASE(2) UBQP_ECASE(3) UBQP_ECASE(4) UBQP_ECASE(5)
        UBQP_ECASE(6) UBQP_ECASE(7) UBQP_ECASE(8) UBQP_ECASE(9) UBQP_ECASE(10) UBQP_ECASE(11)
        UBQP_ECASE(12) UBQP_ECASE(13) UBQP_ECASE(14) UBQP_ECASE(15)
        default: break;
    }
#undef UBQP_ECASE
}
#define UBQP_CCASE(C) \
    case C:           \
        if constexpr (C < NCH) owner_fix_chunk<C, NCH>(K, m, w, kstar & 15, gv, x_new, kfix); \
        break;

// Path relinking (O11, NEXT-4; R19) reuses the ascent loop: variables outside
// D = {j : x_j != y_j} carry keys lowered by kOff = 2^30, below every key in D while
// (2n-1) qmax < 2^21 (checked by ubqp_relink), so the same argmax walks D in gain order
// and the flipped variable leaves D through the owner fix.  The walk takes |D| forced steps
// (moves may worsen f), records the flip order in shared memory and keeps the best strictly
// interior point, rebuilt at the end as x0 xor (first s_best flips).
constexpr int kOff = 1 << 30;
struct RelinkArgs {
    const uint64_t *guides = nullptr;   // [n_guides][W64]; guide of list entry i: i mod n_guides
    int64_t n_guides = 0;
    int32_t *sbest = nullptr;           // [m] step of the best interior point (-1: none)
    int32_t *len = nullptr;             // [m] |D|
};

template <int BLOCK, int NCH, int MINB, bool FULL, bool RELINK>
__global__ void __launch_bounds__(BLOCK, MINB)
ascend_kernel(const int32_t *__restrict__ slots, int max_flips, int n, int n_pad, int q_ld, int W64,
              int64_t k_local, int rank, int world, int shard_b, const int8_t *__restrict__ Q8,
              const int32_t *__restrict__ gains, const int64_t *__restrict__ f_in,
              const uint64_t *__restrict__ Xb, int64_t *__restrict__ f_out,
              int32_t *__restrict__ flips_out, uint64_t *__restrict__ bits_out,
              long long *__restrict__ best_key, const RelinkArgs rl) {
    using A = Asc<BLOCK, NCH>;
    static_assert(A::E <= 128, "local index must fit 7 bits");
    // per-warp winners as one orderable word: (Delta + 2^30) << 32 | ~(j << 1 | x), so a
    // plain unsigned 64-bit max picks the largest gain, then the lowest index
    __shared__ unsigned long long s_win[2][A::NW];
    __shared__ uint32_t s_bits[(A::CHUNK * NCH) / 32];
    __shared__ int s_nd;
    extern __shared__ uint16_t s_seq[];        // RELINK: flip order (n_pad entries)

    const int i = blockIdx.x;
    const int t = threadIdx.x;
    const int lane = t & 31, warp = t >> 5;
    const int64_t s = slots[i];
    if (s < 0 || s >= k_local) {               // invalid slot: reported as flips = -1
        if (t == 0) {
            if (flips_out) flips_out[i] = -1;
            if (f_out) f_out[i] = 0;
            if constexpr (RELINK) {
                if (rl.sbest) rl.sbest[i] = -1;
                if (rl.len) rl.len[i] = -1;
            }
        }
        return;
    }

    int K[NCH][16];
    uint32_t m[NCH][4];
    const int32_t *grow = gains + s * n_pad;
    const uint64_t *xrow = Xb + s * W64;
    const uint64_t *yrow = RELINK ? rl.guides + (i % rl.n_guides) * W64 : nullptr;
    int nd_local = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int j0 = c * A::CHUNK + 16 * t;
        uint32_t bits16 = 0, out16 = 0;        // out16: variables outside D (relinking)
        if (j0 < n) bits16 = static_cast<uint32_t>(xrow[j0 >> 6] >> (j0 & 63)) & 0xFFFFu;
        if constexpr (RELINK) {
            if (j0 < n) {
                const uint32_t d16 = (bits16 ^ static_cast<uint32_t>(yrow[j0 >> 6] >> (j0 & 63))) & 0xFFFFu &
                                     (n - j0 >= 16 ? 0xFFFFu : ((1u << (n - j0)) - 1u));
                nd_local += __popc(d16);
                out16 = ~d16 & 0xFFFFu;
            }
        }
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) m[c][wi] = byte_mask_of_nibble((bits16 >> (4 * wi)) & 15u);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            int4 g = make_int4(0, 0, 0, 0);
            if (j0 < n_pad) g = *reinterpret_cast<const int4 *>(grow + j0 + 4 * q4);
            const int gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int e = 4 * q4 + b;
                const int li = 16 * c + e;
                K[c][e] = (j0 + e < n) ? gg[b] * 256 + 2 * (127 - li) + static_cast<int>((bits16 >> e) & 1u) -
                                             (RELINK && ((out16 >> e) & 1u) ? kOff : 0)
                                       : kPad;
            }
        }
    }
    int nd = 0;
    if constexpr (RELINK) {
        if (t == 0) s_nd = 0;
        __syncthreads();
        if (nd_local) atomicAdd(&s_nd, nd_local);
        __syncthreads();
        nd = s_nd;
    }
    int run = kPad;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int e = 0; e < 16; ++e) run = max(run, K[c][e]);

    const int8_t *qbase = Q8 + 16 * t;        // + kstar*q_ld + c*CHUNK per step
    bool cvalid[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) cvalid[c] = c * A::CHUNK + 16 * t < n_pad;
    int64_t fv = f_in[s];
    int flips = 0;
    int par = 0;
    long long best_f = LLONG_MIN;              // RELINK: best strictly interior point
    int best_s = -1;
    for (;;) {
        // ---- argmax: lane -> warp (max Delta, then min j) -> block
        const int dv = run >> 8;
        const int wv = __reduce_max_sync(0xFFFFFFFFu, dv);
        unsigned cand = 0xFFFFFFFFu;
        if (dv == wv) {
            const int li = 127 - ((run >> 1) & 127);
            const int j = (li >> 4) * A::CHUNK + 16 * t + (li & 15);
            cand = (static_cast<unsigned>(j) << 1) | static_cast<unsigned>(run & 1);
        }
        const unsigned wk = __reduce_min_sync(0xFFFFFFFFu, cand);
        int gv;
        unsigned gk;
        if constexpr (A::NW == 1) {
            gv = wv;
            gk = wk;
        } else {
            if (lane == 0)
                s_win[par][warp] = (static_cast<unsigned long long>(static_cast<unsigned>(wv + (1 << 30))) << 32) |
                                   static_cast<unsigned long long>(~wk);
            __syncthreads();
            unsigned long long best = s_win[par][0];
#pragma unroll
            for (int w2 = 1; w2 < A::NW; ++w2) best = max(best, s_win[par][w2]);
            gv = static_cast<int>(static_cast<unsigned>(best >> 32)) - (1 << 30);
            gk = ~static_cast<unsigned>(best);
            par ^= 1;
        }
        if constexpr (RELINK) {
            if (flips == nd) break;
        } else {
            if (gv <= 0 || flips == max_flips) break;
        }

        // ---- flip k*
        const int kstar = static_cast<int>(gk >> 1);
        const int xk = static_cast<int>(gk & 1u);
        UBQP_DCHECK(kstar >= 0 && kstar < n);
        const int C = xk ? -512 : 512;          // 512 d, d = 1 - 2 x_k*
        fv += gv;
        ++flips;
        if constexpr (RELINK) {
            if (t == 0) s_seq[flips - 1] = static_cast<uint16_t>(kstar);
            if (flips < nd && fv > best_f) {
                best_f = fv;
                best_s = flips;
            }
        }
        constexpr int kfix = RELINK ? kOff : 0;   // k* leaves D
        // 32-bit row offset (kstar * q_ld < 2^31 for n <= 16384): a shorter chain to the row loads
        const uint4 *qrow = reinterpret_cast<const uint4 *>(qbase + static_cast<uint32_t>(kstar) * static_cast<uint32_t>(q_ld));
        uint4 w[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (FULL)      // capacity <= q_ld: every chunk lies in the zero-padded row
                w[c] = __ldg(qrow + c * (A::CHUNK / 16));
            else
                w[c] = cvalid[c] ? __ldg(qrow + c * (A::CHUNK / 16)) : make_uint4(0, 0, 0, 0);
        }
        if (((kstar % A::CHUNK) >> 4) == t) {
            const int x_new = xk ^ 1;
            switch (kstar / A::CHUNK) {
                UBQP_CCASE(0) UBQP_CCASE(1) UBQP_CCASE(2) UBQP_CCASE(3)
                UBQP_CCASE(4) UBQP_CCASE(5) UBQP_CCASE(6) UBQP_CCASE(7)
                default: break;
            }
        }
        // ---- fused update + next argmax.  Per 4 variables: t = w ^ m gives ~q where x = 1;
        // interleave (t_e, m_e) byte pairs and let IDP2A add C t_e - C m_e = C s_e q_e
        // (m_e = -1 where x_e = 1, so the ones' complement is completed exactly).
        const uint32_t a2 = (static_cast<uint32_t>(C) & 0xFFFFu) | (static_cast<uint32_t>(-C) << 16);
        int r0 = kPad, r1 = kPad, r2 = kPad, r3 = kPad;   // 8 independent max chains
        int r4 = kPad, r5 = kPad, r6 = kPad, r7 = kPad;
#pragma unroll
        for (int cc = 0; cc < NCH; ++cc) {
            const int c = NCH - 1 - cc;
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) {
                const uint32_t mw = m[c][wi];
                const uint32_t tq = word_of(w[c], wi) ^ mw;
                int &k0 = K[c][4 * wi + 0];
                int &k1 = K[c][4 * wi + 1];
                int &k2 = K[c][4 * wi + 2];
                int &k3 = K[c][4 * wi + 3];
                const uint32_t blo = __byte_perm(tq, mw, 0x5140);   // t0 m0 t1 m1
                const uint32_t bhi = __byte_perm(tq, mw, 0x7362);   // t2 m2 t3 m3
                k0 = dp2a_lo(a2, blo, k0);
                k1 = dp2a_hi(a2, blo, k1);
                k2 = dp2a_lo(a2, bhi, k2);
                k3 = dp2a_hi(a2, bhi, k3);
                if (c & 1) {
                    if (wi & 2) {
                        r6 = max(r6, max(k0, k1));
                        r7 = max(r7, max(k2, k3));
                    } else {
                        r4 = max(r4, max(k0, k1));
                        r5 = max(r5, max(k2, k3));
                    }
                } else {
                    if (wi & 2) {
                        r2 = max(r2, max(k0, k1));
                        r3 = max(r3, max(k2, k3));
                    } else {
                        r0 = max(r0, max(k0, k1));
                        r1 = max(r1, max(k2, k3));
                    }
                }
            }
        }
        run = max(max(max(r0, r1), max(r2, r3)), max(max(r4, r5), max(r6, r7)));
    }

    // ---- outputs
    if constexpr (RELINK) {
        // x at the best interior step: x0 xor the first best_s flips
        __syncthreads();
        if (bits_out) {
            for (int w2 = t; w2 < W64; w2 += BLOCK) {
                const uint64_t x0w = xrow[w2];
                s_bits[2 * w2] = static_cast<uint32_t>(x0w);
                s_bits[2 * w2 + 1] = static_cast<uint32_t>(x0w >> 32);
            }
            __syncthreads();
            for (int f2 = t; f2 < best_s; f2 += BLOCK) {
                const int j = s_seq[f2];
                atomicXor(&s_bits[j >> 5], 1u << (j & 31));
            }
            __syncthreads();
            for (int w2 = t; w2 < W64; w2 += BLOCK)
                bits_out[static_cast<int64_t>(i) * W64 + w2] =
                    static_cast<uint64_t>(s_bits[2 * w2]) | (static_cast<uint64_t>(s_bits[2 * w2 + 1]) << 32);
        }
        if (t == 0) {
            if (f_out) f_out[i] = best_f;
            if (flips_out) flips_out[i] = flips;
            if (rl.sbest) rl.sbest[i] = best_s;
            if (rl.len) rl.len[i] = nd;
            if (best_key && best_s >= 0) {
                const int64_t g = global_index(s, rank, world, shard_b);
                const long long key = static_cast<long long>(
                    (static_cast<uint64_t>(best_f + (1ll << 40)) << 22) |
                    static_cast<uint64_t>((1ll << 22) - 1 - g));
                atomicMax(best_key, key);
            }
        }
        return;
    }
    if (bits_out) {
        for (int w2 = t; w2 < (A::CHUNK * NCH) / 32; w2 += BLOCK) s_bits[w2] = 0;
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int j0 = c * A::CHUNK + 16 * t;
            uint32_t b16 = 0;
#pragma unroll
            for (int wi = 0; wi < 4; ++wi) b16 |= nibble_of_byte_mask(m[c][wi]) << (4 * wi);
            if (b16) atomicOr(&s_bits[j0 >> 5], b16 << (j0 & 31));
        }
        __syncthreads();
        for (int w2 = t; w2 < W64; w2 += BLOCK)
            bits_out[static_cast<int64_t>(i) * W64 + w2] =
                static_cast<uint64_t>(s_bits[2 * w2]) | (static_cast<uint64_t>(s_bits[2 * w2 + 1]) << 32);
    }
    if (t == 0) {
        if (f_out) f_out[i] = fv;
        if (flips_out) flips_out[i] = flips;
        if (best_key) {
            const int64_t g = global_index(s, rank, world, shard_b);
            const long long key = static_cast<long long>(
                (static_cast<uint64_t>(fv + (1ll << 40)) << 22) |
                static_cast<uint64_t>((1ll << 22) - 1 - g));
            atomicMax(best_key, key);
        }
    }
}
#undef UBQP_CCASE

template <int BLOCK, int NCH>
void launch_inst(Ctx &c, const int32_t *slots, int64_t m, int32_t max_flips, int64_t *f_dev,
                 int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev, const RelinkArgs *rl) {
    const bool full = 16 * BLOCK * NCH <= c.q_ld;
    // register budget ~ 16*NCH keys + 4*NCH masks + 4*NCH loaded words + ~25
    // registers ~ 16*NCH keys + 8*NCH mask/load words + ~30: 168 at NCH = 5
    // 170: 6 CTAs of 64 threads per SM for 96-112 keys (small spills at NCH = 7, measured
    // faster than 5 CTAs); 128 for 80 keys: 8 CTAs, no spills (same-box A/B: n = 5000
    // 1.09 -> 1.40 Gsteps/s; 96 keys at 128 spill 104 B and lose)
    constexpr int kRegs = NCH == 5 ? 128 : (NCH >= 6 ? 170 : 24 * NCH + 48);
    constexpr int kMinBlocks = (65536 / (BLOCK * kRegs)) < 1 ? 1 : 65536 / (BLOCK * kRegs);
    long long *bk = reinterpret_cast<long long *>(best_dev);
    const unsigned grid = static_cast<unsigned>(m);
    if (rl) {
        const size_t seq = static_cast<size_t>(c.n_pad) * sizeof(uint16_t);
        if (full)
            ascend_kernel<BLOCK, NCH, kMinBlocks, true, true><<<grid, BLOCK, seq, c.stream>>>(
                slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
                c.Xb, f_dev, flips_dev, bits_dev, bk, *rl);
        else
            ascend_kernel<BLOCK, NCH, kMinBlocks, false, true><<<grid, BLOCK, seq, c.stream>>>(
                slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
                c.Xb, f_dev, flips_dev, bits_dev, bk, *rl);
        return;
    }
    if (full)
        ascend_kernel<BLOCK, NCH, kMinBlocks, true, false><<<grid, BLOCK, 0, c.stream>>>(
            slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
            c.Xb, f_dev, flips_dev, bits_dev, bk, RelinkArgs{});
    else
        ascend_kernel<BLOCK, NCH, kMinBlocks, false, false><<<grid, BLOCK, 0, c.stream>>>(
            slots, max_flips, c.n, c.n_pad, c.q_ld, c.W64, c.k_local, c.rank, c.world, c.shard_b, c.Q8, c.gains, c.f,
            c.Xb, f_dev, flips_dev, bits_dev, bk, RelinkArgs{});
}

}  // namespace

// Shape: the instantiated (BLOCK, NCH) with the least capacity 16*BLOCK*NCH >= n_pad, ties
// to more variables per thread (64x7 at n = 7000: 98% of the lanes carry a variable; 64x5 at
// n = 5000).  Fewer, fuller threads amortise the per-step argmax exchange (measured at
// config 4: 96x5 306 ms, 64x7 277 ms).  Q8 rows are padded with zeros to this capacity
// (Ctx::q_ld) so the default shape loads every chunk unpredicated.
// UBQP_ASC_CFG="BLOCK,NCH" forces a shape (tuning sweeps, tools/asc_sweep.py).
// Returns 0 on success, 1 if n is outside the instantiated range.
static const int kShapes[][2] = {{32, 1}, {32, 2}, {32, 3}, {32, 4}, {32, 5}, {32, 6}, {32, 7},
                                  {64, 5}, {64, 6}, {64, 7}, {96, 5}, {96, 6}, {96, 7},
                                  {128, 5}, {128, 6}, {128, 7}, {160, 6}, {160, 7}};
// the instantiated shape with the smallest capacity >= n_pad (ties: more variables per thread)
static void default_shape(int np, int &b, int &nch) {
    int best = -1;
    for (int i = 0; i < static_cast<int>(sizeof(kShapes) / sizeof(kShapes[0])); ++i) {
        const int cap = 16 * kShapes[i][0] * kShapes[i][1];
        if (cap < np) continue;
        if (best < 0) { best = i; continue; }
        const int bcap = 16 * kShapes[best][0] * kShapes[best][1];
        if (cap < bcap || (cap == bcap && kShapes[i][1] > kShapes[best][1])) best = i;
    }
    b = kShapes[best][0];
    nch = kShapes[best][1];
}
int ascend_capacity(int n_pad) {
    int b, nch;
    default_shape(n_pad, b, nch);
    return 16 * b * nch;
}

static int launch_walk(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                       int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev, const RelinkArgs *rl) {
    if (m <= 0) return 0;
    const int np = c.n_pad;
    int fb = 0, fn = 0;
    if (const char *env = getenv("UBQP_ASC_CFG")) {
        if (sscanf(env, "%d,%d", &fb, &fn) != 2 || fb * 16 * fn < np) fb = fn = 0;
    }
    int db, dn;   // default shape
    default_shape(np, db, dn);
    if (!fb) { fb = db; fn = dn; }
#define UBQP_ASC(B, N)                                                                          \
    if (fb == B && fn == N) {                                                                   \
        launch_inst<B, N>(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev, rl); \
        ++c.launches;                                                                           \
        return 0;                                                                               \
    }
#define UBQP_ASC_ALL                                                                                  \
    UBQP_ASC(32, 1) UBQP_ASC(32, 2) UBQP_ASC(32, 3) UBQP_ASC(32, 4) UBQP_ASC(32, 5) UBQP_ASC(32, 6)   \
    UBQP_ASC(32, 7) UBQP_ASC(64, 5) UBQP_ASC(64, 6) UBQP_ASC(64, 7) UBQP_ASC(96, 5) UBQP_ASC(96, 6)   \
    UBQP_ASC(96, 7) UBQP_ASC(128, 5) UBQP_ASC(128, 6) UBQP_ASC(128, 7) UBQP_ASC(160, 6)               \
    UBQP_ASC(160, 7)
    UBQP_ASC_ALL
    fb = db;                       // a forced shape that is not instantiated: use the default
    fn = dn;
    UBQP_ASC_ALL
#undef UBQP_ASC_ALL
#undef UBQP_ASC
    return 1;
}

bool ascent_uses_sparse(const Ctx &c) {
    // automatic selection: the dense register kernel everywhere -- the sparse-row kernel was
    // measured slower at every density tried (0.02 .. 0.2, n = 1000 .. 7000; DESIGN.md §7.4')
    if (c.asc_kernel == 2) return true;
    if (c.asc_kernel == 1 || !c.ell || c.n < 2) return false;
    return static_cast<double>(c.nnz) < kSparseAutoDensity * c.n * (c.n - 1.0);
}

int launch_ascend(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                  int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev) {
    if (ascent_uses_sparse(c)) {
        c.asc_last = 2;
        return launch_ascend_sparse(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev);
    }
    // automatic: the warp-per-solution kernel where it measured faster than the CTA kernel
    // (profiles/r02_small_n_kernels.log, 8192 starts): every n_pad in (3584, 7168] (4 KB rows:
    // 1.95 vs 1.44 Gsteps/s at n = 4096) and the 4- and 6-chunk shapes (+3-4% at n = 2048,
    // 3072); the CTA kernel keeps 1-3, 5 and 7 chunks (n = 500: 7.7 vs 6.9, n = 2560: 3.16 vs 2.96)
    const int wch = (c.n_pad + 511) / 512;
    const bool warp_auto = c.n_pad <= ascend_warp_max_n() && (wch >= 8 || wch == 4 || wch == 6);
    if (c.asc_kernel == 3 || (c.asc_kernel == 0 && warp_auto)) {
        c.asc_last = 3;
        return launch_ascend_warp(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev);
    }
    // automatic: 2-4 warps per solution above the one-warp range (n_pad > 7168; measured against
    // the CTA kernel: n = 9000 0.660 vs 0.652, 12000 0.492 vs 0.438, 16000 0.335 vs 0.230 Gsteps/s)
    if (c.asc_kernel == 4 || (c.asc_kernel == 0 && c.n_pad > ascend_warp_max_n())) {
        c.asc_last = 4;
        return launch_ascend_mw(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev);
    }
    c.asc_last = 1;
    return launch_walk(c, slots_dev, m, max_flips, f_dev, flips_dev, bits_dev, best_dev, nullptr);
}

int launch_relink(Ctx &c, const int32_t *slots_dev, int64_t m, const uint64_t *guides_dev, int64_t n_guides,
                  int64_t *f_dev, int32_t *steps_dev, int32_t *sbest_dev, int32_t *len_dev, uint64_t *bits_dev,
                  int64_t *best_dev) {
    RelinkArgs rl;
    rl.guides = guides_dev;
    rl.n_guides = n_guides;
    rl.sbest = sbest_dev;
    rl.len = len_dev;
    return launch_walk(c, slots_dev, m, 0, f_dev, steps_dev, bits_dev, best_dev, &rl);
}

}  // namespace ubqp
