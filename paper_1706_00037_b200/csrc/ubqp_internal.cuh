// ubqp_internal.cuh — handle layout, launch declarations and sm_100a PTX helpers for
// libubqp.so.  Not part of the ABI (include/ubqp.h is).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/ubqp.h"

namespace ubqp {

// ------------------------------------------------------------------ tiling constants
constexpr int kBM = 128;          // eval tile rows (solutions) per CTA: UMMA M
constexpr int kBN = 256;          // eval tile columns (variables j): UMMA N
constexpr int kBK = 128;          // bytes of K (int8 elements) per pipeline stage = one 128B swizzle atom
constexpr int kUmmaK = 32;        // K per tcgen05.mma kind::i8
constexpr int kStages = 4;        // smem pipeline depth
constexpr int kNPadAlign = 128;   // n_pad multiple (K dim of the GEMM)
constexpr int kQRowAlign = kBN;   // Q8 rows padded to a multiple of the N tile
constexpr int kSlices = 4;        // int8 limb planes of the real-Q walk image (28-bit, R20)
constexpr int kMaxLimbs = 10;     // int8 limb planes of the real-Q evaluation image (R22)
constexpr int kMaxPlanes = kMaxLimbs;

// fold modes of the evaluation kernel (eval_tc.cu)
enum { kFoldInt = 0, kFoldPlane = 1, kFoldReal = 2 };

// One B operand of the evaluation GEMM: 1..kMaxPlanes int8 planes of Q (plane s weighs 128^s)
struct Operand {
    int planes = 0;
    bool tri = false;                 // lower triangles: f-only triangular evaluation (NEXT-1)
    CUtensorMap full[kMaxPlanes]{};   // 256-row B boxes (single-CTA kernel)
    CUtensorMap half[kMaxPlanes]{};   // 128-row B boxes (CTA-pair kernel: each CTA half of N)
    const int32_t *diag[kMaxPlanes]{};
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool sticky_cuda = false;
    std::string err;
    int num_sms = 148;

    // instance
    int n = 0, n_pad = 0, q_rows = 0, W64 = 0;
    int q_ld = 0;                // Q8 row stride >= n_pad: the ascent's register capacity (zero tail)
    int8_t *Q8 = nullptr;        // [q_rows][q_ld] row-major, zero padded; row k = column k (Q = Q^t)
    int32_t *diag = nullptr;     // [q_rows]
    int qmax = 0;                // max |Q_ij| of the loaded integer Q
    int8_t *Q8L = nullptr;       // [q_rows][n_pad] lower triangle of Q (row j: Q_ji for i <= j): f-only eval
    Operand op_full, op_tri;     // integer Q: Q8 (gains) and Q8L (f only)
    // sparse rows of the integer Q (NEXT-3): fixed-stride (ELL) rows without the diagonal,
    // entries (j << 8 | (q & 0xFF)), padded with 0xFFFFFFFF to ell_stride (longest row, x32)
    int64_t nnz = 0;             // off-diagonal nonzeros
    int ell_stride = 0;
    uint32_t *ell = nullptr;     // [n][ell_stride]
    int asc_kernel = 0;          // 0 auto, 1 dense CTA, 2 sparse, 3 dense warp, 4 dense multi-warp (UBQP_OPT_ASCENT)
    int asc_last = 0;            // kernel of the last ascend (1 CTA, 2 sparse, 3 warp; UBQP_Q_ASCENT_LAST)
    uint64_t *seed = nullptr;    // [W64] staged diversification seed
    uint64_t *parents = nullptr; // [parents_cap][W64] staged blend parents (host callers)
    int64_t parents_cap = 0;
    uint64_t *guides = nullptr;  // [guides_cap][W64] staged relinking guides (host callers)
    int64_t guides_cap = 0;
    // batch workspace
    int64_t k_max = 0, k_cap_pad = 0, k_local = -1;
    int rank = 0, world = 1;
    int shard_b = 2;             // O10 block size B (UBQP_OPT_SHARD_BLOCK): g = (rank + (i/B) world) B + i%B
    uint64_t *Xb = nullptr;      // [k_max][W64] packed solutions
    int8_t *X8 = nullptr;        // [k_cap_pad][n_pad] expanded 0/1 bytes (GEMM A operand)
    int64_t *f = nullptr;        // [k_max] xQx of the batch
    int32_t *gains = nullptr;    // [k_max][n_pad] 1-flip gains (lazy)
    bool f_valid = false, gains_valid = false;
    int32_t *surv = nullptr;     // [k_max]
    int32_t *blk_count = nullptr;// screen block counts
    int64_t *scratch64 = nullptr;// small device scratch (stats, m, best key)
    // in-kernel fold of the evaluation (eval_tc.cu): row partials, group counters and results
    int32_t *part = nullptr;     // int32 partial row-dots, part_cap elements
    int64_t part_cap = 0;
    unsigned *grp_cnt = nullptr; // [grp_cap] self-resetting arrival counters (last one: groups done)
    int64_t grp_cap = 0;
    int64_t *grp_res = nullptr;  // [grp_cap][4]
    // poll-mode fold (small launches, eval_tc.cu): the same shapes, every word preset to the
    // sentinel 0x80808080 (never a partial) / 0x8080808080808080 and reset by its reader
    int32_t *part_poll = nullptr; // part_cap elements
    int64_t *grp_poll = nullptr;  // [grp_cap][2]
    // ascent outputs scratch
    int64_t *asc_f = nullptr; int32_t *asc_flips = nullptr; uint64_t *asc_bits = nullptr;
    int32_t *asc_slots = nullptr; int32_t *asc_aux = nullptr; int64_t asc_cap = 0;
    // TMA descriptor of the batch (A operand)
    CUtensorMap tmap_X8{};
    bool eval_pair = true;       // UBQP_EVAL_2SM=0 selects the single-CTA kernel
    bool eval_attr_set = false, eval_pair_attr_set = false;   // dynamic-smem opt-in done
    bool sym_eval = true;        // f-only evaluations use the triangular GEMM (UBQP_FULL_EVAL disables)
    // real-valued Q (a4').  Evaluation image (R22): Qw~ = 2^-w_exp sum_s 128^s Lw_s with w_limbs
    // int8 planes, exact for float32 Q and within 2^-32 relative per coefficient otherwise.
    // Walk image (R20): Qt = rint(Q 2^q_exp), 28 bits, as 4 int8 planes (initial gains) and int32
    // rows (the ascent streams them).
    bool real = false;
    int w_exp = 0, w_limbs = 0;
    int8_t *Qw[kMaxLimbs] = {};  // [q_rows][q_ld] full planes (first-derivative row sums)
    int8_t *QwL[kMaxLimbs] = {}; // [q_rows][n_pad] lower triangles (f-only evaluation)
    int32_t *wdiag = nullptr;    // [kMaxLimbs][q_rows] diagonal of each plane
    Operand op_wide;             // QwL planes, tri
    int q_exp = 0;
    int8_t *Qs[kSlices] = {nullptr, nullptr, nullptr, nullptr};   // walk planes [q_rows][q_ld]
    Operand op_walk[kSlices];    // one plane each (EMIT_GAINS launches), zero diagonal
    int32_t *zdiag = nullptr;    // [q_rows] zeros
    int64_t *fs = nullptr;       // [kSlices][k_max] per-walk-plane x^t L_s x
    int64_t *fint = nullptr;     // [k_max] walk image f~28 = sum_s 128^s f_s
    double *freal = nullptr;     // [k_max] f of the evaluation image
    int32_t *Qt = nullptr;
    int qt_ld = 0;
    int32_t *diagt = nullptr;    // [n_pad]
    int64_t *gains64 = nullptr;  // [k_max][n_pad]
    bool gains64_valid = false;
    bool freal_valid = false;
    // re-evaluation workspace of ascended real-Q solutions (their f on the evaluation image)
    int8_t *X8r = nullptr;       // [kReevalRows][n_pad]
    CUtensorMap tmap_X8r{};
    int64_t launches = 0;
};

constexpr int64_t kReevalRows = 8192;   // rows per re-evaluation chunk of ascend_real

// O10: slot i of rank r holds global solution g = (r + floor(i/B) world) B + (i mod B),
// blocks of B consecutive g dealt round robin; B = 1 is plain cyclic sharding.
__host__ __device__ __forceinline__ int64_t global_index(int64_t slot, int rank, int world, int B) {
    return (static_cast<int64_t>(rank) + (slot / B) * world) * B + slot % B;
}

// Shape of one evaluation launch (eval_tc.cu)
constexpr int kMaxSplits = 256;       // K-split table entries per (M tile, plane)
struct EvalShape {
    bool pair;
    int num_n_tiles, num_k_blocks, items_per_group;
    int nsplit;                         // items per (M tile, plane): (N tile, K range) table entries
    uint32_t split_tab[kMaxSplits];     // nt | kb0 << 8 | kb1 << 16, N tile major
    int64_t num_m_tiles, mn_tiles, num_items, num_groups, part_ld, part_elems;
};
struct EvalLaunch {
    const CUtensorMap *tmX = nullptr;  // A operand (batch X8 or the re-evaluation workspace)
    const uint64_t *Xb = nullptr;      // packed bits of the same rows
    int64_t k = 0;
    const Operand *op = nullptr;
    bool emit_gains = false;
    int mode = kFoldInt;
    int64_t *f = nullptr, *f2 = nullptr;
    double *fr = nullptr, *fr2 = nullptr;
    int64_t *stats = nullptr, *stats2 = nullptr;
    int rank = 0, world = 1, shard_b = 1, q_exp = 0;
};

// ------------------------------------------------------------------ launchers (host)
// gen.cu
// parents_dev == nullptr: Glover (O4); else blend with parents_dev[(g mod n_parents)] (O4b)
void launch_glover(Ctx &c, const uint64_t *seed_dev, int64_t t0, int64_t k,
                   const uint64_t *parents_dev = nullptr, int64_t n_parents = 0);
void launch_random(Ctx &c, uint64_t seed, int64_t k);
void launch_expand(Ctx &c, int64_t k);     // Xb -> X8 (after set_batch)
void launch_expand_to(Ctx &c, const uint64_t *bits, int64_t k, int8_t *X8dst);   // any rows -> X8dst
void launch_first_derivative(Ctx &c, uint64_t *bits_dev);   // integer Q8 or the real evaluation planes
// eval_tc.cu
EvalShape eval_shape(const Ctx &c, int64_t k, int planes, bool emit_gains, bool sym);
int launch_eval(Ctx &c, const EvalLaunch &L);   // 1: fold buffers too small (size them first)
// screen.cu
cudaError_t launch_screen(Ctx &c, int64_t k, int64_t t_floor, int64_t *m_dev);   // k <= 0: memset m
cudaError_t launch_screen_real(Ctx &c, int64_t k, double T, int64_t *m_dev);
// ascend_real.cu (R20)
int real_qt_ld(int n_pad);
void launch_gains_combine(Ctx &c, int64_t k, int plane);   // gains64 (+)= gains << 7 plane
int launch_ascend_real(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, double *f_dev,
                       int64_t *fint_dev, int32_t *flips_dev, uint64_t *bits_dev);
// ascend.cu
int ascend_capacity(int n_pad);   // variables covered by the default ascent shape (>= n_pad)
int launch_ascend(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips,
                  int64_t *f_dev, int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev);
// ascend_sparse.cu (NEXT-3): the same walk on CSR rows; 1 if the rows were not built / too large
int launch_ascend_sparse(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                         int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev);
// off-diagonal density below which UBQP_OPT_ASCENT = 0 picks the sparse kernel: 0 = never (it
// was measured slower than the dense kernel at every density tried, DESIGN.md §7.4')
constexpr double kSparseAutoDensity = 0.0;
bool ascent_uses_sparse(const Ctx &c);
// ascend_warp.cu: one warp per solution (n_pad <= ascend_warp_max_n()); 1 if n is out of range
int ascend_warp_max_n();
int launch_ascend_warp(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                       int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev);
// ascend_warp.cu: 2 or 3 warps per solution (n_pad <= ascend_mw_max_n()); 1 if out of range
int ascend_mw_max_n();
int launch_ascend_mw(Ctx &c, const int32_t *slots_dev, int64_t m, int32_t max_flips, int64_t *f_dev,
                     int32_t *flips_dev, uint64_t *bits_dev, int64_t *best_dev);
// path relinking (O11) of batch slots toward guides[i mod n_guides] on the ascent kernel
int launch_relink(Ctx &c, const int32_t *slots_dev, int64_t m, const uint64_t *guides_dev, int64_t n_guides,
                  int64_t *f_dev, int32_t *steps_dev, int32_t *sbest_dev, int32_t *len_dev, uint64_t *bits_dev,
                  int64_t *best_dev);

}  // namespace ubqp

// ------------------------------------------------------------------ device helpers
#ifdef __CUDACC__
// Device-side bounds checks for debug builds (UBQP_NVCC_EXTRA=-DUBQP_DEBUG_CHECKS=1): a failed
// check traps the kernel (the call then returns UBQP_E_CUDA).  compute-sanitizer is closed on
// the GPU pool, so the parity suites run against this build instead (tools/debug_checks.sh).
#ifndef UBQP_DEBUG_CHECKS
#define UBQP_DEBUG_CHECKS 0
#endif
#if UBQP_DEBUG_CHECKS
#define UBQP_DCHECK(cond) \
    do {                  \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define UBQP_DCHECK(cond) ((void)0)
#endif
namespace ubqp {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}

// ---- TMA
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *m, int x, int y,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ---- tcgen05 (cta_group::1)
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, s8 x s8 -> s32
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// 32 lanes x 32 consecutive 32-bit columns: thread (lane) l gets row (lane_base + l).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
}

// ---- CTA pair (cluster of 2, cta_group::2)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_u32(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t *dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// each CTA of the pair loads its half into its own smem; bytes complete on the leader's barrier
__device__ __forceinline__ void tma_load_2d_cg2(void *dst, const CUtensorMap *m, int x, int y,
                                                uint32_t leader_bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(leader_bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mma_i8_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive (when the issued MMAs retire) on the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, rows of 128 B,
// 8-row core-matrix groups 1024 B apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;             // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024u >> 4) << 32;     // SBO
    d |= static_cast<uint64_t>(1u) << 46;             // descriptor version (sm_100)
    d |= static_cast<uint64_t>(2u) << 61;             // SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::i8: D s32, A s8, B s8, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4)                                   // D format: S32
           | (1u << 7)                                 // A: signed 8-bit
           | (1u << 10)                                // B: signed 8-bit
           | (static_cast<uint32_t>(N >> 3) << 17)     // N
           | (static_cast<uint32_t>(M >> 4) << 24);    // M
}

}  // namespace dev
}  // namespace ubqp
#endif
