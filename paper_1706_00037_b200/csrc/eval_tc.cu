// eval_tc.cu — K-EVAL: batched xQx on 5th-generation tensor cores.
//
// Y = X8 · B  (s8 x s8 -> s32, exact), never written to HBM: the accumulator tile lives in
// TMEM and the epilogue folds it immediately into
//     f_k      = sum_j x_kj Y_kj                         (P:24 eq. (P); Appendix A of SURVEY)
//     Delta_kj = Q_jj + 2 (1 - 2 x_kj) Y_kj              (P:53 1-flip gains; UBQP_EMIT_GAINS)
// A = X8 [K x n_pad] K-major; B = an int8 plane of Q [q_rows x n_pad] row-major, which is the
// "N x K, K-major" operand because Q = Q^t (row j = column j).  One launch may run several
// planes (the limb planes of a real-valued Q, a4'): f~ = sum_s 128^s x^t L_s x.
//
// Persistent warp-specialised kernels, one CTA (or CTA pair) per SM:
//   warp 0      : TMA producer (128B-swizzled boxes, smem ring)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  : epilogue (tcgen05.ld 32x32b, thread = row), TMEM double-buffered
//   warp 6      : fold (arrival counters, f and statistics of finished row groups)
// Work item = (plane, M tile, N tile, K split), plane outermost (each plane stays
// L2-resident for its pass), N fastest (the X band in flight is shared through L2).
//
// f and the screening statistics are folded in-kernel (north_star: "the mean/max screening
// reduction fused into the epilogue"): every item's epilogue stores its int32 row partials and
// hands the item to the CTA's fold warp (an mbarrier ring); the fold warp counts the item on its
// 128-row group's counter, and the last item of a group sums the group's partials into f and
// its {sum f, max_key}; the last group to finish reduces all groups into the stats.  Counters
// reset themselves: one launch per evaluation, no memset, no stats kernel.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "ubqp_internal.cuh"

namespace ubqp {
namespace {

constexpr int kThreads = 224;                      // 7 warps: TMA, MMA, 4 epilogue, fold
constexpr int kFoldRing = 4;                       // epilogue -> fold warp hand-off slots
#ifndef UBQP_FOLD_BATCH
#define UBQP_FOLD_BATCH 32
#endif
constexpr int kFoldBatch = UBQP_FOLD_BATCH;        // partial loads in flight per fold lane
constexpr uint32_t kABytes = kBM * kBK;             // 16 KB
constexpr uint32_t kBBytes = kBN * kBK;             // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes; // 48 KB
constexpr uint32_t kTmemCols = 2 * kBN;             // two 128 x 256 s32 accumulators
constexpr size_t kSmemBytes = static_cast<size_t>(kStages) * kStageBytes + 1024 + 512;
constexpr uint32_t kIdesc = dev::idesc_i8(kBM, kBN);

constexpr int kPairStages = 6;
constexpr uint32_t kPairStageBytes = 2 * kABytes;                    // 16 KB A + 16 KB B
constexpr size_t kPairSmemBytes = static_cast<size_t>(kPairStages) * kPairStageBytes + 1024 + 512;
constexpr uint32_t kIdescPair = dev::idesc_i8(2 * kBM, kBN);

// Kernel arguments (one __grid_constant__ block: the B tensor maps of every plane included).
// A/B only (launch-cost experiments): smaller parameter blocks for integer-only builds
#ifndef UBQP_EVAL_PARAM_PLANES
#define UBQP_EVAL_PARAM_PLANES kMaxPlanes
#endif
#ifndef UBQP_EVAL_PARAM_SPLITS
#define UBQP_EVAL_PARAM_SPLITS kMaxSplits
#endif
struct EvalParams {
    CUtensorMap tmX;                      // A = X8
    CUtensorMap tmB[UBQP_EVAL_PARAM_PLANES];          // B per plane (256-row boxes single-CTA, 128-row pair)
    const int32_t *diag[UBQP_EVAL_PARAM_PLANES];      // per-plane diagonal (SYM term, gains)
    int planes;
    int n_pad, W64, num_n_tiles, num_k_blocks;
    int nsplit;                           // items per (M tile, plane) = split_tab entries
    uint32_t split_tab[UBQP_EVAL_PARAM_SPLITS];       // entry o: N tile | kb0 << 8 | kb1 << 16 (host, eval_shape)
    int64_t K, num_m_tiles, num_items;
    const uint64_t *Xb;
    int32_t *gains;                       // EMIT_GAINS target [K][n_pad] (single plane launches)
    int emit_gains;
    // fold
    int32_t *part;                        // [planes][nsplit][part_ld] int32 row partials
    int64_t part_ld;
    unsigned *grp_cnt;                    // [num_groups] arrival counters, then [num_groups]: done
    int items_per_group;
    int64_t num_groups;
    int64_t *grp_res;                     // [num_groups][4]
    int mode;                             // kFoldInt / kFoldPlane / kFoldReal
    int poll;                             // 1: poll-mode fold (fold_item_poll; part / grp_res = the poll buffers)
    int64_t *f, *f2;                      // int f (kFoldInt, kFoldPlane); f2 optional second copy
    double *fr, *fr2;                     // real f (kFoldReal)
    int64_t *stats, *stats2;              // int: {sum, K, max_key, 0}; real: ubqp_stats_real words
    int rank, world, shard_b, q_exp;
};

// Arrival on a fold counter.  The 128 epilogue threads' partial stores are ordered before the
// counter update by the named barrier and the release (cumulative) of the atomic; the last
// arriver's acquire fence orders its reads of the other CTAs' partials after it.  No
// sequentially consistent fence / L1 invalidation in the hot loop (UBQP_FOLD_SYNC=1 selects
// __threadfence() on both sides, for A/B).
#ifndef UBQP_FOLD_SYNC
#define UBQP_FOLD_SYNC 0
#endif
__device__ __forceinline__ unsigned arrive_release(unsigned *ctr) {
#if UBQP_FOLD_SYNC == 1
    __threadfence();
    return atomicAdd(ctr, 1u);
#elif UBQP_FOLD_SYNC == 2
    return atomicAdd(ctr, 1u);   // A/B only: relaxed (no ordering of the partials), measures the fence
#else
    unsigned old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    return old;
#endif
}
__device__ __forceinline__ void acquire_fence() {
#if UBQP_FOLD_SYNC == 1
    __threadfence();
#else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}


// int128 helpers (hi signed, lo unsigned)
constexpr __int128 kI128Min = static_cast<__int128>(static_cast<unsigned __int128>(1) << 127);
struct I128 {
    long long hi;
    unsigned long long lo;
};
__device__ __forceinline__ I128 to_i128(__int128 v) {
    return {static_cast<long long>(v >> 64), static_cast<unsigned long long>(v)};
}
__device__ __forceinline__ __int128 from_i128(long long hi, unsigned long long lo) {
    return (static_cast<__int128>(hi) << 64) | static_cast<__int128>(lo);
}
// correctly rounded int128 -> binary64: the top 64 significant bits with a sticky bit in the
// lsb round to 53 bits exactly as the full value would (cvt.rn.f64.u64 rounds to nearest even)
__device__ __forceinline__ double i128_to_double(__int128 v) {
    const bool neg = v < 0;
    const unsigned __int128 a = neg ? static_cast<unsigned __int128>(-(v + 1)) + 1u : static_cast<unsigned __int128>(v);
    const unsigned long long hi = static_cast<unsigned long long>(a >> 64);
    double d;
    if (hi == 0) {
        d = __ull2double_rn(static_cast<unsigned long long>(a));
    } else {
        const int sh = 64 - __clzll(static_cast<long long>(hi));
        unsigned long long top = static_cast<unsigned long long>(a >> sh);
        const unsigned __int128 low = a & ((static_cast<unsigned __int128>(1) << sh) - 1u);
        if (low != 0) top |= 1ull;
        d = ldexp(__ull2double_rn(top), sh);
    }
    return neg ? -d : d;
}

#ifndef UBQP_EVAL_TRACE
#define UBQP_EVAL_TRACE 0      // 1: %globaltimer stamps per CTA at the pipeline's milestones (debug)
#endif
#if UBQP_EVAL_TRACE
__device__ unsigned long long g_evtrace[512][16];
__device__ __forceinline__ void ev_stamp(int slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 512) g_evtrace[blockIdx.x][slot] = t;
}
#define EV_STAMP(s) ev_stamp(s)
#else
#define EV_STAMP(s) ((void)0)
#endif

// ---------------------------------------------------------------- fold (last arriver per group)
// A dedicated fold warp (warp 6) runs this for every item of its CTA, after the four epilogue
// warps stored their partials and arrived on the item's ring barrier -- so the counter round
// trip and the occasional fold never sit on the epilogue's critical path (the epilogue must
// keep pace with the MMAs).  The last arriver of a 128-row group sums the group's partials
// into f and its {sum f, max_key} (or int128 {sum f~, max f~}); the last group overall
// reduces every group into the statistics.
__device__ __forceinline__ void warp_i128_reduce(__int128 &sm, __int128 &mx, bool &have) {
    for (int o = 16; o > 0; o >>= 1) {
        const I128 a = to_i128(sm), b = to_i128(mx);
        const long long sh = __shfl_xor_sync(0xffffffffu, a.hi, o);
        const unsigned long long sl = __shfl_xor_sync(0xffffffffu, a.lo, o);
        const long long mh = __shfl_xor_sync(0xffffffffu, b.hi, o);
        const unsigned long long ml = __shfl_xor_sync(0xffffffffu, b.lo, o);
        const int oh = __shfl_xor_sync(0xffffffffu, have ? 1 : 0, o);
        sm += from_i128(sh, sl);
        const __int128 om = from_i128(mh, ml);
        if (oh && (!have || om > mx)) mx = om;
        have = have || oh;
    }
}

// ---------------------------------------------------------------- poll-mode fold (small launches)
// When every item of a launch is resident at once (items <= CTA pairs: the paper's Table 1
// shape, K = 1000), the counter chain above is the launch's tail (the arrival
// atomic with its release/acquire fences, then the partials' round trip, twice).  Here every
// partial word is its own flag instead: the buffers hold the sentinel kPollSent32 (0x80808080;
// |partial| <= 256 (2n 127 + 127) < 2^31 - 2^26 at n <= 16384, so it is never a partial) and
// ONE fold warp per 128-row group -- the CTA that ran the group's split 0 -- polls the group's
// partials with L2-only copies (cp.async.cg: every lane's pieces in flight at once) until no
// word is the sentinel, folds f and {sum f, max_key} as above, and puts the sentinel back.
// The group results are flagged the same way (0x8080808080808080: sum f and the key never take
// it) and polled by group 0's folder, which writes the statistics.  No atomics, no fences:
// each word is read only after its own value arrived.  Progress: a spinning fold warp blocks
// no other warp (one item per CTA, so the epilogue never waits on the fold ring), and at most
// one spinning CTA per group stays resident while the others finish their items and exit.
constexpr int kPollSent32 = static_cast<int>(0x80808080u);
constexpr long long kPollSent64 = static_cast<long long>(0x8080808080808080ull);
#ifndef UBQP_POLL_LIMIT
#define UBQP_POLL_LIMIT (1u << 26)   // polls before trapping (seconds): a broken launch fails loudly
#endif

__device__ __forceinline__ bool poll_has_sent(const int4 &t) {
    return t.x == kPollSent32 || t.y == kPollSent32 || t.z == kPollSent32 || t.w == kPollSent32;
}

// stage nb 16-byte pieces (stride ld4 int4) from L2 into shared memory until none holds the
// sentinel; returns with the pieces in sfold[32 u + lane]
__device__ __forceinline__ void poll_pieces(const int4 *ptr0, int64_t ld4, int nb, int lane, int4 *sfold) {
    const uint32_t sdst = dev::smem_u32(sfold) + 16u * lane;
    unsigned want = nb >= 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);   // pieces still to (re)load
    for (unsigned tries = 0;; ++tries) {
        const int4 *ptr = ptr0;
        for (int u = 0; u < nb; ++u, ptr += ld4)
            if ((want >> u) & 1u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst + 512u * u), "l"(ptr) : "memory");
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        unsigned again = 0;
        for (int u = 0; u < nb; ++u)
            if (((want >> u) & 1u) && poll_has_sent(sfold[32 * u + lane])) again |= 1u << u;
        want = again;
        if (__all_sync(0xFFFFFFFFu, want == 0u)) return;
        if (tries > UBQP_POLL_LIMIT) __trap();
    }
}

template <bool SYM>
__device__ __forceinline__ void fold_item_poll(const EvalParams &p, int64_t group, int lane, int4 *sfold) {
    const int64_t row0 = group * 128 + 4 * lane;
    UBQP_DCHECK(p.mode == kFoldInt && p.planes == 1 && group < p.num_groups && row0 + 3 < p.part_ld);
    const int nsplit = p.nsplit;
    const int64_t ld4 = p.part_ld / 4;
    long long sacc[4] = {0, 0, 0, 0};
    int4 *base = reinterpret_cast<int4 *>(p.part + row0);
    const int4 sent = make_int4(kPollSent32, kPollSent32, kPollSent32, kPollSent32);
    for (int s0 = 0; s0 < nsplit; s0 += kFoldBatch) {
        const int nb = min(kFoldBatch, nsplit - s0);
        int4 *ptr = base + static_cast<int64_t>(s0) * ld4;
        poll_pieces(ptr, ld4, nb, lane, sfold);
        for (int u = 0; u < nb; ++u) {
            const int4 t = sfold[32 * u + lane];
            sacc[0] += t.x;
            sacc[1] += t.y;
            sacc[2] += t.z;
            sacc[3] += t.w;
            __stcg(ptr + static_cast<int64_t>(u) * ld4, sent);   // re-arm for the next launch
        }
    }
    if (lane == 0) EV_STAMP(15);
    long long isum = 0, ikey = -1;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t row = row0 + q;
        if (row >= p.K) continue;
        const long long fsum = sacc[q];
        p.f[row] = fsum;
        if (p.f2) p.f2[row] = fsum;
        const unsigned r32 = static_cast<unsigned>(row), b32 = static_cast<unsigned>(p.shard_b);
        const long long g = p.world == 1 ? static_cast<long long>(row)
                                         : (static_cast<long long>(p.rank) + (r32 / b32) * static_cast<long long>(p.world)) * b32 + r32 % b32;
        const long long key = static_cast<long long>((static_cast<unsigned long long>(fsum + (1ll << 40)) << 22) |
                                                     static_cast<unsigned long long>((1ll << 22) - 1 - g));
        isum += fsum;
        ikey = max(ikey, key);
    }
    for (int o = 16; o > 0; o >>= 1) {
        isum += __shfl_xor_sync(0xffffffffu, isum, o);
        ikey = max(ikey, __shfl_xor_sync(0xffffffffu, ikey, o));
    }
    if (lane == 0) {
        EV_STAMP(11);
        __stcg(reinterpret_cast<longlong2 *>(p.grp_res) + group, make_longlong2(isum, ikey));
    }
    if (group != 0) return;
    // group 0's folder: every group's {sum f, max_key} -> the statistics
    const int ng = static_cast<int>(p.num_groups);
    long long S = 0, M = -1;
    const longlong2 sent2 = make_longlong2(kPollSent64, kPollSent64);
    for (int g0 = 0; g0 < ng; g0 += 32 * kFoldBatch) {
        // piece u of lane = group g0 + 32 u + lane (16 bytes each); out-of-range lanes re-read group 0
        const int nb = min(kFoldBatch, (ng - g0 + 31) / 32);
        const uint32_t sdst = dev::smem_u32(sfold) + 16u * lane;
        unsigned want = 0;
        for (int u = 0; u < nb; ++u)
            if (g0 + 32 * u + lane < ng) want |= 1u << u;
        for (unsigned tries = 0;; ++tries) {
            for (int u = 0; u < nb; ++u)
                if ((want >> u) & 1u)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst + 512u * u),
                                 "l"(reinterpret_cast<const longlong2 *>(p.grp_res) + g0 + 32 * u + lane) : "memory");
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
            unsigned again = 0;
            for (int u = 0; u < nb; ++u) {
                const longlong2 v = reinterpret_cast<const longlong2 *>(sfold)[32 * u + lane];
                if (((want >> u) & 1u) && (v.x == kPollSent64 || v.y == kPollSent64)) again |= 1u << u;
            }
            want = again;
            if (__all_sync(0xFFFFFFFFu, want == 0u)) break;
            if (tries > UBQP_POLL_LIMIT) __trap();
        }
        for (int u = 0; u < nb; ++u) {
            const int g = g0 + 32 * u + lane;
            if (g >= ng) continue;
            const longlong2 v = reinterpret_cast<const longlong2 *>(sfold)[32 * u + lane];
            S += v.x;
            M = max(M, v.y);
            __stcg(reinterpret_cast<longlong2 *>(p.grp_res) + g, sent2);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        M = max(M, __shfl_xor_sync(0xffffffffu, M, o));
    }
    if (lane == 0) {
        EV_STAMP(13);
        const long long out[4] = {S, static_cast<long long>(p.K), M, 0};
        for (int i = 0; i < 4; ++i) {
            p.stats[i] = out[i];
            if (p.stats2) p.stats2[i] = out[i];
        }
    }
}

#ifndef UBQP_FOLD_DEBUG
#define UBQP_FOLD_DEBUG 0   // A/B only: 1 = no fold at all
#endif
template <bool SYM>
__device__ __forceinline__ void fold_item(const EvalParams &p, int64_t group, int lane, int4 *sfold) {
#if UBQP_FOLD_DEBUG == 1
    return;
#endif
    unsigned last = 0;
    if (lane == 0) {
        const unsigned old = arrive_release(&p.grp_cnt[group]);
        last = old + 1u == static_cast<unsigned>(p.items_per_group) ? 1u : 0u;
        if (last) acquire_fence();
    }
    if (lane == 0) EV_STAMP(10);
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    if (lane == 0) EV_STAMP(14);
    if (lane == 0) p.grp_cnt[group] = 0u;              // self-reset for the next launch
#if UBQP_FOLD_DEBUG == 3
    return;                                            // A/B only: counters without the fold work
#endif
    // lane owns rows group*128 + 4 lane .. +3: one 16-byte load per (plane, item), all of a
    // plane's loads independent (8 in flight), accumulated plane by plane (Horner, base 128)
    long long isum = 0, ikey = -1;
    __int128 rsum = 0, rmax = 0;
    bool rhave = false;
    const int64_t row0 = group * 128 + 4 * lane;
    UBQP_DCHECK(group < p.num_groups && row0 + 3 < p.part_ld);
    __int128 acc[4] = {0, 0, 0, 0};
    long long fs[4] = {0, 0, 0, 0};
    const int nsplit = p.nsplit;
    const int64_t ld4 = p.part_ld / 4;
    for (int pl = p.planes - 1; pl >= 0; --pl) {
        long long sacc[4] = {0, 0, 0, 0};
        const int4 *base = reinterpret_cast<const int4 *>(p.part + static_cast<int64_t>(pl) * nsplit * p.part_ld + row0);
        // batches of 32 independent loads: one round trip for up to 32 partials per row (every
        // split-table entry owns >= 1 K block, so every slot is written)
        for (int s0 = 0; s0 < nsplit; s0 += kFoldBatch) {
            // every lane copies its own 16-byte pieces into shared memory (LDGSTS: no registers,
            // so all of them are in flight at once -- register loads let ptxas interleave the sums
            // and serialise the round trips), waits for its own group and reads them back
            const int4 *ptr = base + static_cast<int64_t>(s0) * ld4;
            const uint32_t sdst = dev::smem_u32(sfold) + 16u * lane;
            const int nb = min(kFoldBatch, nsplit - s0);
            for (int u = 0; u < nb; ++u) {
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst + 512u * u), "l"(ptr) : "memory");
                ptr += ld4;
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
            for (int u = 0; u < nb; ++u) {             // shared-memory latency only
                const int4 t = sfold[32 * u + lane];
                sacc[0] += t.x;
                sacc[1] += t.y;
                sacc[2] += t.z;
                sacc[3] += t.w;
            }
        }
        if (lane == 0) EV_STAMP(15);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            acc[q] = acc[q] * 128 + sacc[q];
            fs[q] = sacc[q];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int64_t row = row0 + q;
        if (row >= p.K) continue;
        const long long fsum = fs[q];
        if (p.mode == kFoldPlane) {
            p.f[row] = fsum;
        } else if (p.mode == kFoldInt) {
            p.f[row] = fsum;
            if (p.f2) p.f2[row] = fsum;
            const unsigned r32 = static_cast<unsigned>(row), b32 = static_cast<unsigned>(p.shard_b);
            const long long g = p.world == 1 ? static_cast<long long>(row)     // 32-bit form of global_index
                                             : (static_cast<long long>(p.rank) + (r32 / b32) * static_cast<long long>(p.world)) * b32 + r32 % b32;
            const long long key = static_cast<long long>((static_cast<unsigned long long>(fsum + (1ll << 40)) << 22) |
                                                         static_cast<unsigned long long>((1ll << 22) - 1 - g));
            isum += fsum;
            ikey = max(ikey, key);
        } else {
            const double fr = ldexp(i128_to_double(acc[q]), -p.q_exp);
            p.fr[row] = fr;
            if (p.fr2) p.fr2[row] = fr;
            rsum += acc[q];
            if (!rhave || acc[q] > rmax) rmax = acc[q];
            rhave = true;
        }
    }
    if (lane == 0) EV_STAMP(11);
    if (p.mode == kFoldPlane) return;
    if (p.mode == kFoldInt) {
        for (int o = 16; o > 0; o >>= 1) {
            isum += __shfl_xor_sync(0xffffffffu, isum, o);
            ikey = max(ikey, __shfl_xor_sync(0xffffffffu, ikey, o));
        }
        if (lane == 0) {
            p.grp_res[4 * group + 0] = isum;
            p.grp_res[4 * group + 1] = ikey;
        }
    } else {
        warp_i128_reduce(rsum, rmax, rhave);
        if (!rhave) rmax = kI128Min;                   // no solution in this group
        if (lane == 0) {
            const I128 a = to_i128(rsum), b = to_i128(rmax);
            p.grp_res[4 * group + 0] = a.hi;
            p.grp_res[4 * group + 1] = static_cast<long long>(a.lo);
            p.grp_res[4 * group + 2] = b.hi;
            p.grp_res[4 * group + 3] = static_cast<long long>(b.lo);
        }
    }
    // the last group overall folds every group's result into the statistics
    __syncwarp();
    last = 0;
    if (lane == 0) {
        const unsigned old = arrive_release(p.grp_cnt + p.num_groups);
        last = old + 1u == static_cast<unsigned>(p.num_groups) ? 1u : 0u;
        if (last) acquire_fence();
        EV_STAMP(12);
    }
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    if (p.mode == kFoldInt) {
        long long S = 0, M = -1;
#pragma unroll 8
        for (int64_t g = lane; g < p.num_groups; g += 32) {
            S += __ldcg(p.grp_res + 4 * g);
            M = max(M, static_cast<long long>(__ldcg(p.grp_res + 4 * g + 1)));
        }
        for (int o = 16; o > 0; o >>= 1) {
            S += __shfl_xor_sync(0xffffffffu, S, o);
            M = max(M, __shfl_xor_sync(0xffffffffu, M, o));
        }
        if (lane == 0) {
            EV_STAMP(13);
            const long long out[4] = {S, static_cast<long long>(p.K), M, 0};
            for (int i = 0; i < 4; ++i) {
                p.stats[i] = out[i];
                if (p.stats2) p.stats2[i] = out[i];
            }
            p.grp_cnt[p.num_groups] = 0u;
        }
    } else {
        __int128 S = 0, M = kI128Min;
        bool H = false;
#pragma unroll 4
        for (int64_t g = lane; g < p.num_groups; g += 32) {
            S += from_i128(__ldcg(p.grp_res + 4 * g), static_cast<unsigned long long>(__ldcg(p.grp_res + 4 * g + 1)));
            const __int128 m2 =
                from_i128(__ldcg(p.grp_res + 4 * g + 2), static_cast<unsigned long long>(__ldcg(p.grp_res + 4 * g + 3)));
            if (!H || m2 > M) M = m2;
            H = true;
        }
        warp_i128_reduce(S, M, H);
        if (lane == 0) {
            const I128 a = to_i128(S), b = to_i128(M);
            const long long out[6] = {a.hi, static_cast<long long>(a.lo), static_cast<long long>(p.K), b.hi,
                                      static_cast<long long>(b.lo), static_cast<long long>(static_cast<unsigned>(p.q_exp))};
            for (int i = 0; i < 6; ++i) {
                p.stats[i] = out[i];
                if (p.stats2) p.stats2[i] = out[i];
            }
            p.grp_cnt[p.num_groups] = 0u;
        }
    }
}

// Epilogue of one 128-row x 256-column accumulator (thread = row): drains TMEM 32 columns at a
// time and folds  f_k += sum_j x_kj Y_kj  (or, triangular: x_kj (2 Y_kj - Q_jj), the Q_jj term
// only in the K split that owns the diagonal) and, with gains, stores
// Delta_kj = Q_jj + 2 (1 - 2 x_kj) Y_kj.  Returns the row's int32 partial of f.
// The tile's diagonal slice (256 ints) is staged per warp in shared memory (sdiag, one
// coalesced round trip) and the row's 256 solution bits are loaded up front: no memory
// latency inside the TMEM drain loop (what bounds small-K launches).
// Stage the tile's diagonal slice and load the row's 256 solution bits: independent of the
// MMAs, so it is issued BEFORE the wait for the accumulator (measured at K = 1000: the loads'
// round trip otherwise sits between TMEM-full and the drain).
template <bool SYM>
__device__ __forceinline__ void epilogue_stage(int64_t row, bool row_ok, int n0, int W64,
                                               const uint64_t *__restrict__ Xb, const int32_t *__restrict__ diag,
                                               int emit_gains, bool with_diag, int32_t *sdiag, int lane,
                                               uint64_t (&xw)[4]) {
    const bool need_diag = SYM ? with_diag : (emit_gains != 0);
    __syncwarp();                                      // the previous tile's reads of sdiag are done
    if (need_diag) {
        const int4 *dg = reinterpret_cast<const int4 *>(diag + n0);
        reinterpret_cast<int4 *>(sdiag)[lane] = __ldg(dg + lane);
        reinterpret_cast<int4 *>(sdiag)[lane + 32] = __ldg(dg + lane + 32);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int w = (n0 >> 6) + q;
        xw[q] = (row_ok && w < W64) ? Xb[row * W64 + w] : 0ull;
    }
    __syncwarp();
}

// One 32-column chunk of the drain (thread = row): f partial, and with gains the gain stores.
template <bool SYM>
__device__ __forceinline__ void epilogue_chunk(const uint32_t (&v)[32], int c, int32_t &partial, int64_t row,
                                               bool row_ok, int n0, int n_pad, int32_t *__restrict__ gains,
                                               int emit_gains, bool with_diag, const int32_t *sdiag,
                                               const uint64_t (&xw)[4]) {
    const int col0 = n0 + c * 32;
    const int q = c >> 1;                          // select, not an indexed (local) array
    const uint64_t wq = q == 0 ? xw[0] : (q == 1 ? xw[1] : (q == 2 ? xw[2] : xw[3]));
    const uint32_t bits = static_cast<uint32_t>(wq >> (32 * (c & 1)));
    const int4 *dg = reinterpret_cast<const int4 *>(sdiag + c * 32);
    if constexpr (SYM) {
        if (with_diag) {
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
                const int4 d = dg[i4];
                const int dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = 4 * i4 + e;
                    partial += ((bits >> i) & 1u) ? 2 * static_cast<int32_t>(v[i]) - dd[e] : 0;
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) partial += ((bits >> i) & 1u) ? 2 * static_cast<int32_t>(v[i]) : 0;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) partial += ((bits >> i) & 1u) ? static_cast<int32_t>(v[i]) : 0;
        if (emit_gains && row_ok && col0 < n_pad) {
            int4 *gp = reinterpret_cast<int4 *>(gains + row * n_pad + col0);
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {
                const int4 d = dg[i4];
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

template <bool SYM>
__device__ __forceinline__ int32_t epilogue_tile(uint32_t t_row, int64_t row, bool row_ok, int n0, int n_pad,
                                                 int32_t *__restrict__ gains, int emit_gains, bool with_diag,
                                                 const int32_t *sdiag, const uint64_t (&xw)[4]) {
    using namespace dev;
    int32_t partial = 0;
    // double-buffered drain: chunk c + 1 is read from TMEM while chunk c is folded
    // (tcgen05.wait::ld waits for every outstanding load, so the loads alternate buffers)
    uint32_t va[32], vb[32];
    tmem_ld_32x32b_x32(t_row, va);
#pragma unroll 1
    for (int c = 0; c < kBN / 32; c += 2) {
        tmem_wait_ld();
        tmem_ld_32x32b_x32(t_row + static_cast<uint32_t>((c + 1) * 32), vb);
        epilogue_chunk<SYM>(va, c, partial, row, row_ok, n0, n_pad, gains, emit_gains, with_diag, sdiag, xw);
        tmem_wait_ld();
        if (c + 2 < kBN / 32) tmem_ld_32x32b_x32(t_row + static_cast<uint32_t>((c + 2) * 32), va);
        epilogue_chunk<SYM>(vb, c + 1, partial, row, row_ok, n0, n_pad, gains, emit_gains, with_diag, sdiag, xw);
    }
    return partial;
}

// Work item -> (plane, M tile, split-table entry = (N tile, K block range)), plane outermost,
// then M tile, then N tile.  f is linear in Y, so the partial row-dots of K splits add up in the
// fold; the -Q_jj term of SYM goes with the split owning kb 0.
struct Item {
    int plane, mt, nt, sidx, kb0, kb1;
};
template <bool SYM>
__device__ __forceinline__ Item decode_item(const EvalParams &p, int64_t item) {
    Item it;
    const int64_t per_plane = p.num_m_tiles * p.nsplit;
    it.plane = static_cast<int>(item / per_plane);
    const int64_t r = item - static_cast<int64_t>(it.plane) * per_plane;
    it.mt = static_cast<int>(r / p.nsplit);
    it.sidx = static_cast<int>(r - static_cast<int64_t>(it.mt) * p.nsplit);
    const uint32_t e = p.split_tab[it.sidx];
    it.nt = static_cast<int>(e & 0xFFu);
    it.kb0 = static_cast<int>((e >> 8) & 0xFFu);
    it.kb1 = static_cast<int>(e >> 16);
    UBQP_DCHECK(it.nt < p.num_n_tiles && it.kb0 < it.kb1 && it.kb1 <= p.num_k_blocks && it.plane < p.planes &&
                it.sidx < p.nsplit);
    return it;
}
__device__ __forceinline__ int64_t split_index(const EvalParams &p, const Item &it) {
    return static_cast<int64_t>(it.plane) * p.nsplit + it.sidx;
}

// ---------------------------------------------------------------- single-CTA kernel (M = 128)
template <bool SYM>
__global__ void __launch_bounds__(kThreads, 1) eval_tc_kernel(const __grid_constant__ EvalParams p) {
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
    uint64_t *ffull = tempty + 2;             // epilogue -> fold warp (4 warp arrivals)
    uint64_t *fempty = ffull + kFoldRing;     // fold warp -> epilogue (1 arrival)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(fempty + kFoldRing);
    __shared__ __align__(16) int32_t s_diag[4 * kBN];   // per epilogue warp: the tile's diagonal slice
    __shared__ int4 s_fold[kFoldBatch * 32];             // fold warp: one batch of staged partials

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
        for (int r = 0; r < kFoldRing; ++r) {
            mbar_init(&ffull[r], 4);
            mbar_init(&fempty[r], 1);
        }
        fence_mbar_init();
        tma_prefetch(&p.tmX);
        for (int pl = 0; pl < p.planes; ++pl) tma_prefetch(&p.tmB[pl]);
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
            for (int64_t item = blockIdx.x; item < p.num_items; item += gridDim.x) {
                const Item it = decode_item<SYM>(p, item);
                for (int kb = it.kb0; kb < it.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&full[stage], kStageBytes);
                    tma_load_2d(sA + stage * kABytes, &p.tmX, kb * kBK, it.mt * kBM, &full[stage], pol_x);
                    tma_load_2d(sB + stage * kBBytes, &p.tmB[it.plane], kb * kBK, it.nt * kBN, &full[stage], pol_q);
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
            for (int64_t item = blockIdx.x; item < p.num_items; item += gridDim.x) {
                const Item it = decode_item<SYM>(p, item);
                if (it.kb0 == it.kb1) continue;
                mbar_wait(&tempty[acc], acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
                for (int kb = it.kb0; kb < it.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * kABytes));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * kBBytes));
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k) {
                        // +32 bytes along K inside the 128B swizzle atom = +2 in the >>4 field
                        mma_i8(d_tmem, adesc + 2u * k, bdesc + 2u * k, kIdesc, (kb != it.kb0 || k != 0) ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);   // frees the smem slot when these MMAs retire
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
                mma_commit(&tfull[acc]);         // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
            }
        }
    } else if (warp == 6) {
        // ---------------- fold warp: counts each item's arrival for its group, folds the last
        int fslot = 0;
        uint32_t fphase = 0;
        for (int64_t item = blockIdx.x; item < p.num_items; item += gridDim.x) {
            const Item it = decode_item<SYM>(p, item);
            if (it.kb0 == it.kb1) continue;
            mbar_wait(&ffull[fslot], fphase);
            fold_item<SYM>(p, it.mt, lane, s_fold);
            __syncwarp();
            if (lane == 0) mbar_arrive(&fempty[fslot]);
            if (++fslot == kFoldRing) { fslot = 0; fphase ^= 1u; }
        }
    } else {
        // ---------------- epilogue: warp w may read TMEM lanes 32*(w%4) .. +31
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        int fslot = 0;
        uint32_t fphase = 0;
        for (int64_t item = blockIdx.x; item < p.num_items; item += gridDim.x) {
            const Item it = decode_item<SYM>(p, item);
            if (it.kb0 == it.kb1) continue;
            const int64_t row = static_cast<int64_t>(it.mt) * kBM + row_in_tile;
            const bool row_ok = row < p.K;
            uint64_t xw[4];
            epilogue_stage<SYM>(row, row_ok, it.nt * kBN, p.W64, p.Xb, p.diag[it.plane], p.emit_gains, it.kb0 == 0,
                                s_diag + quarter * kBN, lane, xw);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) EV_STAMP(5);
            const int32_t partial = epilogue_tile<SYM>(
                tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kBN), row,
                row_ok, it.nt * kBN, p.n_pad, p.gains, p.emit_gains, it.kb0 == 0, s_diag + quarter * kBN, xw);
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
            mbar_wait(&fempty[fslot], fphase ^ 1u);           // the fold warp released this slot
            UBQP_DCHECK(row < p.part_ld && split_index(p, it) < static_cast<int64_t>(p.planes) * p.nsplit);
            p.part[split_index(p, it) * p.part_ld + row] = partial;
            __syncwarp();
            if (lane == 0) mbar_arrive(&ffull[fslot]);        // release: the warp's partials are stored
            if (++fslot == kFoldRing) { fslot = 0; fphase ^= 1u; }
            if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------- CTA-pair kernel (M = 256)
// cta_group::2: a cluster of two CTAs on one TPC computes a 256 x 256 tile with M = 256 MMAs
// issued by the leader; each CTA stages its 128 rows of X and its 128 rows of B per K block
// (32 KB per stage instead of 48 KB), so the shared-memory and L2 traffic per MAC halves for
// B.  Accumulators: each CTA's TMEM holds its 128 rows x 256 columns (two buffers).  Each
// CTA's epilogue folds its own 128-row group.
template <bool SYM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
eval_tc_pair_kernel(const __grid_constant__ EvalParams p) {
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
    uint64_t *ffull = tempty + 2;             // epilogue -> fold warp (4 warp arrivals)
    uint64_t *fempty = ffull + kFoldRing;     // fold warp -> epilogue (1 arrival)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(fempty + kFoldRing);
    __shared__ __align__(16) int32_t s_diag[4 * kBN];   // per epilogue warp: the tile's diagonal slice
    __shared__ int4 s_fold[kFoldBatch * 32];             // fold warp: one batch of staged partials

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        EV_STAMP(0);
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);           // the leader's expect_tx; both CTAs' bytes land here
            mbar_init(&empty[s], 1);          // multicast commit of the leader's MMAs
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);          // multicast commit
            mbar_init(&tempty[a], 8);         // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        for (int r = 0; r < kFoldRing; ++r) {
            mbar_init(&ffull[r], 4);          // this CTA's 4 epilogue warps stored their partials
            mbar_init(&fempty[r], 1);         // this CTA's fold warp is done with the slot
        }
        fence_mbar_init();
        tma_prefetch(&p.tmX);
        for (int pl = 0; pl < p.planes; ++pl) tma_prefetch(&p.tmB[pl]);
    }
    if (warp == 1) tmem_alloc_cg2(tmem_slot, kTmemCols);
    tc_fence_before();
    cluster_sync();                           // barriers of both CTAs initialised, TMEM allocated
    // programmatic dependent launch (launch_eval): the next kernel on the stream may launch now.
    // Only this kernel triggers early, so a predecessor still running is another evaluation,
    // which writes f, the statistics, the gains and the fold buffers but never X8, the Q planes
    // or the diagonals: the TMA producer and the MMA issuer (reads of X8 / Q, TMEM writes) start
    // at once, the epilogue and fold warps wait for the predecessor's completion (and memory)
    // before their first global access.  No-ops when launched without the attribute.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (warp >= 2) asm volatile("griddepcontrol.wait;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) EV_STAMP(1);

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- TMA producer (both CTAs: own half of A and of B)
            const uint64_t pol_q = policy_evict_last();
            const uint64_t pol_x = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t item = cid; item < p.num_items; item += ncl) {
                const Item it = decode_item<SYM>(p, item);
                const int m0 = it.mt * (2 * kBM) + static_cast<int>(rank) * kBM;
                const int n0 = it.nt * kBN + static_cast<int>(rank) * (kBN / 2);
                for (int kb = it.kb0; kb < it.kb1; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * kPairStageBytes);
                    const uint32_t fb = mapa_u32(&full[stage], 0);
                    tma_load_2d_cg2(sA + stage * kABytes, &p.tmX, kb * kBK, m0, fb, pol_x);
                    tma_load_2d_cg2(sB + stage * kABytes, &p.tmB[it.plane], kb * kBK, n0, fb, pol_q);
                    if (++stage == kPairStages) { stage = 0; phase ^= 1u; }
                }
            }
            EV_STAMP(2);
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ---------------- MMA issuer (leader only): M = 256 across the pair
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t item = cid; item < p.num_items; item += ncl) {
                const Item it = decode_item<SYM>(p, item);
                if (it.kb0 == it.kb1) continue;
                mbar_wait(&tempty[acc], acc_phase ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
                for (int kb = it.kb0; kb < it.kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (kb == it.kb0 && item == cid) EV_STAMP(3);
                    const uint64_t adesc = umma_desc_sw128(smem_u32(sA + stage * kABytes));
                    const uint64_t bdesc = umma_desc_sw128(smem_u32(sB + stage * kABytes));
#pragma unroll
                    for (int k = 0; k < kBK / kUmmaK; ++k)
                        mma_i8_cg2(d_tmem, adesc + 2u * k, bdesc + 2u * k, kIdescPair,
                                   (kb != it.kb0 || k != 0) ? 1u : 0u);
                    mma_commit_pair(&empty[stage]);
                    if (++stage == kPairStages) { stage = 0; phase ^= 1u; }
                }
                mma_commit_pair(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
            }
            EV_STAMP(4);
        }
    } else if (warp == 6) {
        // ---------------- fold warp (each CTA: its own group)
        int fslot = 0;
        uint32_t fphase = 0;
        for (int64_t item = cid; item < p.num_items; item += ncl) {
            const Item it = decode_item<SYM>(p, item);
            if (it.kb0 == it.kb1) continue;
            mbar_wait(&ffull[fslot], fphase);
            if (lane == 0) EV_STAMP(7);
            if (p.poll) {
                if (it.sidx == 0) fold_item_poll<SYM>(p, static_cast<int64_t>(it.mt) * 2 + rank, lane, s_fold);
            } else {
                fold_item<SYM>(p, static_cast<int64_t>(it.mt) * 2 + rank, lane, s_fold);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&fempty[fslot]);
            if (++fslot == kFoldRing) { fslot = 0; fphase ^= 1u; }
        }
        if (lane == 0) EV_STAMP(8);
    } else {
        // ---------------- epilogue (both CTAs: their own 128 rows)
        const int quarter = warp & 3;
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t tempty_leader0 = mapa_u32(&tempty[0], 0);
        const uint32_t tempty_leader1 = mapa_u32(&tempty[1], 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        int fslot = 0;
        uint32_t fphase = 0;
        for (int64_t item = cid; item < p.num_items; item += ncl) {
            const Item it = decode_item<SYM>(p, item);
            if (it.kb0 == it.kb1) continue;
            const int64_t group = static_cast<int64_t>(it.mt) * 2 + rank;
            const int64_t row = group * kBM + row_in_tile;
            const bool row_ok = row < p.K;
            uint64_t xw[4];
            epilogue_stage<SYM>(row, row_ok, it.nt * kBN, p.W64, p.Xb, p.diag[it.plane], p.emit_gains, it.kb0 == 0,
                                s_diag + quarter * kBN, lane, xw);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) EV_STAMP(5);
            const int32_t partial = epilogue_tile<SYM>(
                tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * kBN), row,
                row_ok, it.nt * kBN, p.n_pad, p.gains, p.emit_gains, it.kb0 == 0, s_diag + quarter * kBN, xw);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
            mbar_wait(&fempty[fslot], fphase ^ 1u);           // the fold warp released this slot
            UBQP_DCHECK(row < p.part_ld && split_index(p, it) < static_cast<int64_t>(p.planes) * p.nsplit);
            p.part[split_index(p, it) * p.part_ld + row] = partial;
            __syncwarp();
            if (lane == 0) mbar_arrive(&ffull[fslot]);        // release: the warp's partials are stored
            if (++fslot == kFoldRing) { fslot = 0; fphase ^= 1u; }
            if (++acc == 2) { acc = 0; acc_phase ^= 1u; }
        }
        if (warp == 2 && lane == 0) EV_STAMP(6);
    }

    tc_fence_before();
    cluster_sync();                           // all MMAs retired, both epilogues done
    if (threadIdx.x == 0) EV_STAMP(9);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_cg2(tmem_base, kTmemCols);
    }
}

}  // namespace

#if UBQP_EVAL_TRACE
// debug builds only: copy the per-CTA stamps of the last pair launch (512 x 16 ns timestamps)
extern "C" int ubqp_debug_eval_trace(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_evtrace, sizeof(g_evtrace)) == cudaSuccess ? 0 : 1;
}
#endif

// Shapes of a launch (host): items, groups, the K-split table and the partial buffer.
// Items of one (M tile, plane) are the entries of the split table: N tile nt (its K blocks:
// all of them, or, triangular, the kbs(nt) = min(num_k_blocks, 2 (nt + 1)) blocks of rows < 256
// (nt + 1)) cut into s(nt) K ranges.  s(nt) = 1 unless an f-only CTA-pair launch has fewer
// tiles than CTA pairs; then the K blocks are BALANCED over the pairs: the least T >= 2 with
// num_m_tiles planes sum_nt ceil(kbs(nt) / T) <= pairs, s(nt) = ceil(kbs(nt) / T), so every
// pair runs one item of <= T blocks (round 2's uniform power-of-two splits left the largest
// tiles with 2x the blocks and some pairs with two items; measured at K = 1000: the MMA phase's
// tail was 6.7 us against a 3.8 us median).  UBQP_KSPLIT = s forces s(nt) = min(s, kbs(nt)).
EvalShape eval_shape(const Ctx &c, int64_t k, int planes, bool emit_gains, bool sym) {
    EvalShape s;
    s.pair = c.eval_pair;
    s.num_n_tiles = (c.n + kBN - 1) / kBN;
    s.num_k_blocks = c.n_pad / kBK;
    const int rows = s.pair ? 2 * kBM : kBM;
    s.num_m_tiles = (k + rows - 1) / rows;
    s.mn_tiles = s.num_m_tiles * s.num_n_tiles;
    static const int forced = [] {
        const char *e = getenv("UBQP_KSPLIT");
        return e ? atoi(e) : 0;
    }();
    int kbs[64];
    int total = 0;
    for (int nt = 0; nt < s.num_n_tiles; ++nt) {
        kbs[nt] = sym ? std::min(s.num_k_blocks, (nt + 1) * (kBN / kBK)) : s.num_k_blocks;
        total += kbs[nt];
    }
    int T = 1 << 30;                                   // max K blocks per item (no split)
    const int64_t pairs = c.num_sms / 2;
    if (s.pair && !emit_gains && s.mn_tiles * planes < pairs) {
        const int64_t per = pairs / (s.num_m_tiles * planes);   // items per (M tile, plane)
        for (T = 2; T < s.num_k_blocks; ++T) {
            int64_t cnt = 0;
            for (int nt = 0; nt < s.num_n_tiles; ++nt) cnt += (kbs[nt] + T - 1) / T;
            if (cnt <= per) break;
        }
    }
    s.nsplit = 0;
    for (int nt = 0; nt < s.num_n_tiles; ++nt) {
        int parts = (kbs[nt] + T - 1) / T;
        if (s.pair && !emit_gains && forced > 0) parts = std::min(forced, kbs[nt]);
        parts = std::max(1, std::min(parts, kMaxSplits - s.nsplit - (s.num_n_tiles - 1 - nt)));
        for (int q = 0; q < parts; ++q) {
            const int kb0 = q * kbs[nt] / parts, kb1 = (q + 1) * kbs[nt] / parts;
            s.split_tab[s.nsplit++] = static_cast<uint32_t>(nt) | (static_cast<uint32_t>(kb0) << 8) |
                                      (static_cast<uint32_t>(kb1) << 16);
        }
    }
    s.num_items = s.num_m_tiles * planes * s.nsplit;
    s.items_per_group = planes * s.nsplit;
    s.num_groups = s.num_m_tiles * (s.pair ? 2 : 1);
    s.part_ld = s.num_groups * kBM;
    s.part_elems = static_cast<int64_t>(planes) * s.nsplit * s.part_ld;
    return s;
}

int launch_eval(Ctx &c, const EvalLaunch &L) {
    if (L.k <= 0) return 0;
    const bool sym = L.op->tri && !L.emit_gains;
    const EvalShape s = eval_shape(c, L.k, L.op->planes, L.emit_gains, sym);
    if (s.part_elems > c.part_cap || s.num_groups + 1 > c.grp_cap) return 1;   // caller sizes first
    EvalParams p{};
    p.tmX = *L.tmX;
    for (int i = 0; i < L.op->planes; ++i) {
        p.tmB[i] = s.pair ? L.op->half[i] : L.op->full[i];
        p.diag[i] = L.op->diag[i];
    }
    p.planes = L.op->planes;
    p.n_pad = c.n_pad;
    p.W64 = c.W64;
    p.num_n_tiles = s.num_n_tiles;
    p.num_k_blocks = s.num_k_blocks;
    p.nsplit = s.nsplit;
    for (int o = 0; o < s.nsplit; ++o) p.split_tab[o] = s.split_tab[o];
    p.K = L.k;
    p.num_m_tiles = s.num_m_tiles;
    p.num_items = s.num_items;
    p.Xb = L.Xb;
    p.gains = L.emit_gains ? c.gains : nullptr;
    p.emit_gains = L.emit_gains ? 1 : 0;
    p.part = c.part;
    p.part_ld = s.part_ld;
    p.grp_cnt = c.grp_cnt;
    p.items_per_group = s.items_per_group;
    p.num_groups = s.num_groups;
    p.grp_res = c.grp_res;
    p.mode = L.mode;
    // poll-mode fold: CTA-pair launches of integer f whose items all run at once (one per pair)
    static const bool poll_ok = [] {
        const char *e = getenv("UBQP_EVAL_POLL");
        return !(e && e[0] == '0');
    }();
    if (poll_ok && s.pair && L.mode == kFoldInt && L.op->planes == 1 && s.num_items <= c.num_sms / 2 &&
        c.part_poll && c.grp_poll) {
        p.poll = 1;
        p.part = c.part_poll;
        p.grp_res = c.grp_poll;
    }
    p.f = L.f;
    p.f2 = L.f2;
    p.fr = L.fr;
    p.fr2 = L.fr2;
    p.stats = L.stats;
    p.stats2 = L.stats2;
    p.rank = L.rank;
    p.world = L.world;
    p.shard_b = L.shard_b;
    p.q_exp = L.q_exp;
    if (s.pair) {
        if (!c.eval_pair_attr_set) {   // per handle (= per device): the attribute is per device context
            cudaFuncSetAttribute(eval_tc_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kPairSmemBytes));
            cudaFuncSetAttribute(eval_tc_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kPairSmemBytes));
            c.eval_pair_attr_set = true;
        }
        const int64_t pairs = s.num_items < c.num_sms / 2 ? s.num_items : c.num_sms / 2;
        // programmatic stream serialization: the launch overlaps the predecessor's tail (its
        // exiting CTAs free SMs for this one's prologue); the kernel's griddepcontrol.wait keeps
        // every memory access after the predecessor completed.  UBQP_EVAL_PDL=0: plain launch.
        static const bool pdl = [] {
            const char *e = getenv("UBQP_EVAL_PDL");
            return !(e && e[0] == '0');
        }();
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kPairSmemBytes;
        cfg.stream = c.stream;
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        auto go = [&]() {
            return sym ? cudaLaunchKernelEx(&cfg, eval_tc_pair_kernel<true>, p)
                       : cudaLaunchKernelEx(&cfg, eval_tc_pair_kernel<false>, p);
        };
        if (go() != cudaSuccess && cfg.numAttrs) {   // a stream without programmatic launch: plain
            cudaGetLastError();
            cfg.numAttrs = 0;
            go();                                    // errors reach the caller's CK_LAUNCH
        }
    } else {
        if (!c.eval_attr_set) {
            cudaFuncSetAttribute(eval_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemBytes));
            cudaFuncSetAttribute(eval_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemBytes));
            c.eval_attr_set = true;
        }
        const int grid = static_cast<int>(s.num_items < c.num_sms ? s.num_items : c.num_sms);
        if (sym)
            eval_tc_kernel<true><<<grid, kThreads, kSmemBytes, c.stream>>>(p);
        else
            eval_tc_kernel<false><<<grid, kThreads, kSmemBytes, c.stream>>>(p);
    }
    ++c.launches;
    return 0;
}

}  // namespace ubqp
