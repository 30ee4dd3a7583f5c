// eval_tc.cu — K-EVAL: batched xQx on 5th-generation tensor cores.
//
// Y = X8 · Q8  (s8 x s8 -> s32, exact), never written to HBM: the accumulator tile lives
// in TMEM and the epilogue folds it immediately into
//     f_k      = sum_j x_kj Y_kj                         (P:24 eq. (P); Appendix A of SURVEY)
//     Delta_kj = Q_jj + 2 (1 - 2 x_kj) Y_kj              (P:53 1-flip gains; UBQP_EMIT_GAINS)
// A = X8 [K x n_pad] K-major; B = Q8 [q_rows x n_pad] row-major, which is the "N x K,
// K-major" operand because Q = Q^t (row j of Q8 = column j of Q).
//
// Persistent warp-specialised kernel, one CTA per SM:
//   warp 0      : TMA producer (128B-swizzled 128x128 A and 256x128 B boxes, kStages ring)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=32)
//   warps 2..5  : epilogue (tcgen05.ld 32x32b -> f partial / gains), TMEM double-buffered
// Tiles are ordered n-fastest so the ~5 X bands in flight are shared through L2 by all
// N tiles and Q (49 MB at n = 7000) stays L2-resident.
#include <climits>

#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

constexpr int kThreads = 192;
constexpr uint32_t kABytes = kBM * kBK;             // 16 KB
constexpr uint32_t kBBytes = kBN * kBK;             // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes; // 48 KB
constexpr uint32_t kTmemCols = 2 * kBN;             // two 128 x 256 s32 accumulators
constexpr size_t kSmemBytes = static_cast<size_t>(kStages) * kStageBytes + 1024 + 256;
constexpr uint32_t kIdesc = dev::idesc_i8(kBM, kBN);

// Epilogue of one 128-row x 256-column accumulator (thread = row): drains TMEM 32 columns at a
// time and folds  f_k += sum_j x_kj Y_kj  (or, triangular: x_kj (2 Y_kj - Q_jj), the Q_jj term
// only in the K split that owns the diagonal) and, with gains, stores
// Delta_kj = Q_jj + 2 (1 - 2 x_kj) Y_kj.  Returns the row's int32 partial of f.
template <bool SYM>
__device__ __forceinline__ int32_t epilogue_tile(uint32_t t_row, int64_t row, bool row_ok, int n0, int W64,
                                                 int n_pad, const uint64_t *__restrict__ Xb,
                                                 const int32_t *__restrict__ diag, int32_t *__restrict__ gains,
                                                 int emit_gains, bool with_diag) {
    using namespace dev;
    int32_t partial = 0;
#pragma unroll 1
    for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + static_cast<uint32_t>(c * 32), v);
        tmem_wait_ld();
        const int col0 = n0 + c * 32;
        uint32_t bits = 0;
        if (row_ok && (col0 >> 6) < W64)
            bits = static_cast<uint32_t>(Xb[row * W64 + (col0 >> 6)] >> (col0 & 63));
        if constexpr (SYM) {
            const int4 *dg = reinterpret_cast<const int4 *>(diag + col0);
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
                const int4 d = __ldg(dg + i4);
                const int dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = 4 * i4 + e;
                    partial += ((bits >> i) & 1u) ? 2 * static_cast<int32_t>(v[i]) - (with_diag ? dd[e] : 0) : 0;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) partial += ((bits >> i) & 1u) ? static_cast<int32_t>(v[i]) : 0;
            if (emit_gains && row_ok && col0 < n_pad) {
                const int4 *dg = reinterpret_cast<const int4 *>(diag + col0);
                int4 *gp = reinterpret_cast<int4 *>(gains + row * n_pad + col0);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {
                    const int4 d = __ldg(dg + i4);
                    int o[4];
                    const int dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int i = 4 * i4 + e;
                        const int y2 = 2 * static_cast<int32_t>(v[i]);
                        o[e] = dd[e] + (((bits >> i) & 1u) ? -y2 : y2);
                    }
                    __stcs(gp + i4, make_int4(o[0], o[1], o[2], o[3]));   // streaming: keep X/Q in L2
                }
            }
        }
    }
    return partial;
}

// SYM (f only, NEXT-1 of SURVEY §8(f)): B = the lower triangle of Q (row j keeps Q_ji, i <= j),
// so tile column block J needs only K blocks covering rows i < 256(J+1): ~(n+256)/(2n) of the
// MMAs.  f = sum_j x_j (2 Y^U_j - Q_jj) with Y^U_j = sum_{i<=j} x_i Q_ij  (Q = Q^t).
template <bool SYM>
__global__ void __launch_bounds__(kThreads, 1)
eval_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQ,
               int64_t K, int n_pad, int W64, int num_n_tiles, int num_k_blocks, int64_t num_tiles,
               const uint64_t *__restrict__ Xb, const int32_t *__restrict__ diag,
               int64_t *__restrict__ f, int32_t *__restrict__ gains, int emit_gains) {
    using namespace dev;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~static_cast<uintptr_t>(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + kStages * kABytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageBytes);
    uint64_t *empty = full + kStages;
    uint64_t *tfull = empty + kStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        fence_mbar_init();
        tma_prefetch(&tmX);
        tma_prefetch(&tmQ);
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer
            const uint64_t pol_q = policy_evict_last();
            const uint64_t pol_x = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int m0 = static_cast<int>(tile / num_n_tiles) * kBM;
                const int nt = static_cast<int>(tile % num_n_tiles);
                const int n0 = nt * kBN;
                const int kbs = SYM ? min(num_k_blocks, (nt + 1) * (kBN / kBK)) : num_k_blocks;
                for (int kb = 0; kb < kbs; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&full[stage], kStageBytes);
                    tma_load_2d(sA + stage * kABytes, &tmX, kb * kBK, m0, &full[stage], pol_x);
                    tma_load_2d(sB + stage * kBBytes, &tmQ, kb * kBK, n0, &full[stage], pol_q);
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (one thread issues for the whole CTA)
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
                const int nt = static_cast<int>(tile % num_n_tiles);
                const int kbs = SYM ? min(num_k_blocks, (nt + 1) * (kBN / kBK)) : num_k_blocks;
                for (int kb = 0; kb < kbs; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * kABytes));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * kBBytes));
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k) {
                        // +32 bytes along K inside the 128B swizzle atom = +2 in the >>4 field
                        mma_i8(d_tmem, adesc + 2u * k, bdesc + 2u * k, kIdesc,
                               (kb | k) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);   // frees the smem slot when these MMAs retire
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
                mma_commit(&tfull[acc]);         // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
            }
        }
    } else {
        // ---------------- epilogue: warp w may read TMEM lanes 32*(w%4) .. +31
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int64_t m0 = (tile / num_n_tiles) * kBM;
            const int n0 = static_cast<int>(tile % num_n_tiles) * kBN;
            const int64_t row = m0 + row_in_tile;
            const bool row_ok = row < K;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int32_t partial = epilogue_tile<SYM>(
                tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kBN),
                row, row_ok, n0, W64, n_pad, Xb, diag, gains, emit_gains, true);
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            if (row_ok)
                atomicAdd(reinterpret_cast<unsigned long long *>(f + row),
                          static_cast<unsigned long long>(static_cast<int64_t>(partial)));
            if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------- CTA-pair variant
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with M = 256 MMAs
// issued by the leader; each CTA stages its 128 rows of X and its 128 rows of Q per K block
// (32 KB per stage instead of 48 KB), so the shared-memory and L2 traffic per MAC halves for
// B.  Accumulators: each CTA's TMEM holds its 128 rows x 256 columns (two buffers).
constexpr int kPairStages = 6;
constexpr uint32_t kPairStageBytes = 2 * kABytes;                    // 16 KB A + 16 KB B
constexpr size_t kPairSmemBytes = static_cast<size_t>(kPairStages) * kPairStageBytes + 1024 + 256;
constexpr uint32_t kIdescPair = dev::idesc_i8(2 * kBM, kBN);

// Work item = (M tile of 256 rows, N tile of 256 columns, K split).  f-only launches with
// fewer tiles than CTA pairs split K (f is linear in Y, so the partial row-dots of the splits
// add up in the int64 atomics; the -Q_jj term of SYM goes with split 0).
struct PairTile {
    int mt, nt, kb0, kb1;
};
template <bool SYM>
__device__ __forceinline__ PairTile pair_tile(int64_t tile, int num_n_tiles, int num_k_blocks, int ksplit) {
    PairTile t;
    const int64_t mn = tile / ksplit;
    const int ks = static_cast<int>(tile - mn * ksplit);
    t.mt = static_cast<int>(mn / num_n_tiles);
    t.nt = static_cast<int>(mn - static_cast<int64_t>(t.mt) * num_n_tiles);
    const int kbs = SYM ? min(num_k_blocks, (t.nt + 1) * (kBN / kBK)) : num_k_blocks;
    t.kb0 = ks * kbs / ksplit;
    t.kb1 = (ks + 1) * kbs / ksplit;
    return t;
}

template <bool SYM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
eval_tc_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmQh,
                    int64_t K, int n_pad, int W64, int num_n_tiles, int num_k_blocks, int64_t num_tiles,
                    const uint64_t *__restrict__ Xb, const int32_t *__restrict__ diag,
                    int64_t *__restrict__ f, int32_t *__restrict__ gains, int emit_gains, int ksplit) {
    using namespace dev;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~static_cast<uintptr_t>(1023));
    uint8_t *sA = smem;
    uint8_t *sB = smem + kPairStages * kABytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kPairStages * kPairStageBytes);
    uint64_t *empty = full + kPairStages;
    uint64_t *tfull = empty + kPairStages;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);           // the leader's expect_tx; both CTAs' bytes land here
            mbar_init(&empty[s], 1);          // multicast commit of the leader's MMAs
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);          // multicast commit
            mbar_init(&tempty[a], 8);         // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        fence_mbar_init();
        tma_prefetch(&tmX);
        tma_prefetch(&tmQh);
    }
    if (warp == 1) tmem_alloc_cg2(tmem_slot, kTmemCols);
    tc_fence_before();
    cluster_sync();                           // barriers of both CTAs initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs: own half of A and of B)
            const uint64_t pol_q = policy_evict_last();
            const uint64_t pol_x = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
                const PairTile pt = pair_tile<SYM>(tile, num_n_tiles, num_k_blocks, ksplit);
                if (pt.kb0 == pt.kb1) continue;
                const int m0 = pt.mt * (2 * kBM) + static_cast<int>(rank) * kBM;
                const int n0 = pt.nt * kBN + static_cast<int>(rank) * (kBN / 2);
                for (int kb = pt.kb0; kb < pt.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kPairStageBytes);
                    const uint32_t fb = mapa_u32(&full[stage], 0);
                    tma_load_2d_cg2(sA + stage * kABytes, &tmX, kb * kBK, m0, fb, pol_x);
                    tma_load_2d_cg2(sB + stage * kABytes, &tmQh, kb * kBK, n0, fb, pol_q);
                    if (++stage == kPairStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ---------------- MMA issuer (leader only): M = 256 across the pair
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
                const PairTile pt = pair_tile<SYM>(tile, num_n_tiles, num_k_blocks, ksplit);
                if (pt.kb0 == pt.kb1) continue;
                mbar_wait(&tempty[acc], acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
                for (int kb = pt.kb0; kb < pt.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * kABytes));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * kABytes));
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k)
                        mma_i8_cg2(d_tmem, adesc + 2u * k, bdesc + 2u * k, kIdescPair,
                                   (kb != pt.kb0 || k != 0) ? 1u : 0u);
                    mma_commit_pair(&empty[stage]);
                    if (++stage == kPairStages) { stage = 0; phase ^= 1u; }
                }
                mma_commit_pair(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
            }
        }
    } else {
        // ---------------- epilogue (both CTAs: their own 128 rows)
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t tempty_leader0 = mapa_u32(&tempty[0], 0);
        const uint32_t tempty_leader1 = mapa_u32(&tempty[1], 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int64_t tile = cid; tile < num_tiles; tile += ncl) {
            const PairTile pt = pair_tile<SYM>(tile, num_n_tiles, num_k_blocks, ksplit);
            if (pt.kb0 == pt.kb1) continue;
            const bool with_diag = pt.kb0 == 0;
            const int64_t m0 = static_cast<int64_t>(pt.mt) * (2 * kBM) + rank * kBM;
            const int n0 = pt.nt * kBN;
            const int64_t row = m0 + row_in_tile;
            const bool row_ok = row < K;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int32_t partial = epilogue_tile<SYM>(
                tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kBN),
                row, row_ok, n0, W64, n_pad, Xb, diag, gains, emit_gains, with_diag);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
            if (row_ok)
                atomicAdd(reinterpret_cast<unsigned long long *>(f + row),
                          static_cast<unsigned long long>(static_cast<int64_t>(partial)));
            if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
    }

    tc_fence_before();
    cluster_sync();                           // all MMAs retired, both epilogues done
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2(tmem_base, kTmemCols);
    }
}


// ---------------------------------------------------------------- batch statistics
__global__ void __launch_bounds__(1024) stats_kernel(const int64_t *__restrict__ f, int64_t K,
                                                     int rank, int world,
                                                     int64_t *__restrict__ out) {
    __shared__ int64_t s_sum[32], s_key[32];
    int64_t sum = 0, key = -1;
    for (int64_t i = threadIdx.x; i < K; i += blockDim.x) {
        const int64_t v = f[i];
        sum += v;
        const int64_t g = static_cast<int64_t>(rank) + i * world;
        const int64_t k = static_cast<int64_t>(
            (static_cast<uint64_t>(v + (1ll << 40)) << 22) |
            static_cast<uint64_t>((1ll << 22) - 1 - g));
        key = k > key ? k : key;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const int64_t other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
    }
    if ((threadIdx.x & 31) == 0) {
        s_sum[threadIdx.x >> 5] = sum;
        s_key[threadIdx.x >> 5] = key;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t S = 0, M = -1;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            S += s_sum[w];
            M = s_key[w] > M ? s_key[w] : M;
        }
        out[0] = S;
        out[1] = K;
        out[2] = M;
        out[3] = 0;
    }
}


}  // namespace

void launch_eval_tc(Ctx &c, int64_t k, bool emit_gains, int plane, int64_t *f_out, bool sym) {
    const CUtensorMap *tmap_q = plane >= 0 ? &c.tmap_Qs[plane] : nullptr;
    if (k <= 0) return;
    if (!c.eval_attr_set) {   // per handle (= per device): the attribute is per device context
        cudaFuncSetAttribute(eval_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemBytes));
        cudaFuncSetAttribute(eval_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemBytes));
        c.eval_attr_set = true;
    }
    const int num_n_tiles = (c.n + kBN - 1) / kBN;
    const int num_k_blocks = c.n_pad / kBK;
    const bool use_sym = sym && !emit_gains;
    if (c.eval_pair) {
        if (!c.eval_pair_attr_set) {
            cudaFuncSetAttribute(eval_tc_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kPairSmemBytes));
            cudaFuncSetAttribute(eval_tc_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kPairSmemBytes));
            c.eval_pair_attr_set = true;
        }
        const int64_t mn_tiles = ((k + 2 * kBM - 1) / (2 * kBM)) * num_n_tiles;
        // f-only launches too small to fill the pairs twice split K (<= 8 ways)
        int ksplit = 1;
        if (!emit_gains)
            while (ksplit < 8 && mn_tiles * ksplit < c.num_sms && num_k_blocks >= 4 * ksplit) ksplit *= 2;
        const int64_t num_tiles = mn_tiles * ksplit;
        const int64_t pairs = num_tiles < c.num_sms / 2 ? num_tiles : c.num_sms / 2;
        const CUtensorMap &tq = use_sym ? c.tmap_Q8L_h : (plane >= 0 ? c.tmap_Qs_h[plane] : c.tmap_Q8_h);
        if (use_sym)
            eval_tc_pair_kernel<true><<<static_cast<unsigned>(2 * pairs), kThreads, kPairSmemBytes, c.stream>>>(
                c.tmap_X8, tq, k, c.n_pad, c.W64, num_n_tiles, num_k_blocks, num_tiles, c.Xb, c.diag,
                f_out ? f_out : c.f, nullptr, 0, ksplit);
        else
            eval_tc_pair_kernel<false><<<static_cast<unsigned>(2 * pairs), kThreads, kPairSmemBytes, c.stream>>>(
                c.tmap_X8, tq, k, c.n_pad, c.W64, num_n_tiles, num_k_blocks, num_tiles, c.Xb, c.diag,
                f_out ? f_out : c.f, emit_gains ? c.gains : nullptr, emit_gains ? 1 : 0, ksplit);
        ++c.launches;
        return;
    }
    const int64_t num_m_tiles = (k + kBM - 1) / kBM;
    const int64_t num_tiles = num_m_tiles * num_n_tiles;
    const int grid = static_cast<int>(num_tiles < c.num_sms ? num_tiles : c.num_sms);
    if (use_sym)
        eval_tc_kernel<true><<<grid, kThreads, kSmemBytes, c.stream>>>(
            c.tmap_X8, c.tmap_Q8L, k, c.n_pad, c.W64, num_n_tiles, num_k_blocks, num_tiles, c.Xb,
            c.diag, f_out ? f_out : c.f, nullptr, 0);
    else
        eval_tc_kernel<false><<<grid, kThreads, kSmemBytes, c.stream>>>(
            c.tmap_X8, tmap_q ? *tmap_q : c.tmap_Q8, k, c.n_pad, c.W64, num_n_tiles, num_k_blocks,
            num_tiles, c.Xb, c.diag, f_out ? f_out : c.f, emit_gains ? c.gains : nullptr, emit_gains ? 1 : 0);
    ++c.launches;
}

// ---------------------------------------------------------------- real-valued Q (a4')
// f~_k = sum_s 128^s f_s,k (exact int64), f_k = 2^-q_exp f~_k; stats over the integer image:
// {sum f~ as int128 (hi, lo), count, max f~} so ranks can reduce them exactly.
__global__ void __launch_bounds__(1024) combine_real_kernel(const int64_t *__restrict__ fs, int64_t k_max,
                                                            int64_t K, int q_exp,
                                                            int64_t *__restrict__ fint,
                                                            double *__restrict__ freal,
                                                            int64_t *__restrict__ out) {
    __shared__ unsigned long long s_lo[32];
    __shared__ long long s_hi[32];
    __shared__ long long s_max[32];
    __int128 sum = 0;
    long long mx = LLONG_MIN;
    for (int64_t i = threadIdx.x; i < K; i += blockDim.x) {
        int64_t v = 0;
#pragma unroll
        for (int s = kSlices - 1; s >= 0; --s) v = v * 128 + fs[s * k_max + i];
        fint[i] = v;
        freal[i] = ldexp(static_cast<double>(v), -q_exp);
        sum += v;
        mx = v > mx ? v : mx;
    }
    // reduce the int128 sum as (hi, lo) halves with carries
    unsigned long long lo = static_cast<unsigned long long>(sum);
    long long hi = static_cast<long long>(sum >> 64);
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
        const long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
        const unsigned long long nlo = lo + olo;
        hi = hi + ohi + (nlo < lo ? 1 : 0);
        lo = nlo;
        const long long omx = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = omx > mx ? omx : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
        s_max[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long L = 0;
        long long H = 0, M = LLONG_MIN;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
            const unsigned long long nl = L + s_lo[w];
            H = H + s_hi[w] + (nl < L ? 1 : 0);
            L = nl;
            M = s_max[w] > M ? s_max[w] : M;
        }
        out[0] = H;
        out[1] = static_cast<int64_t>(L);
        out[2] = K;
        out[3] = M;
    }
}

void launch_combine_real(Ctx &c, int64_t k, int64_t *stats_dev) {
    combine_real_kernel<<<1, 1024, 0, c.stream>>>(c.fs, c.k_max, k, c.q_exp, c.fint, c.freal, stats_dev);
    ++c.launches;
}

void launch_stats(Ctx &c, int64_t k, int64_t *stats_dev) {
    stats_kernel<<<1, 1024, 0, c.stream>>>(c.f, k, c.rank, c.world, stats_dev);
    ++c.launches;
}

}  // namespace ubqp
