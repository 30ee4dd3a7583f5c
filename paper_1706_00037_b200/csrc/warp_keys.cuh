// warp_keys.cuh — device helpers shared by the warp-per-solution ascent (ascend_warp.cu) and the
// multi-warp ascent (ascend_mw.cu): the dp2a key updates, 3-input max/min, the per-lane cp.async
// row staging and the uniform jump table that adds to one register-resident key.
#pragma once
#include <cstdint>

namespace ubqp {
namespace {

// volatile keeps the updates in source order in the PTX (word by word, each followed by its
// max/min); the SASS order is ptxas's own (see the chain restart in the loop).  The measured
// bench build uses the volatile form; UBQP_WARP_VOLATILE=0 is the plain-asm A/B variant.
#ifndef UBQP_WARP_VOLATILE
#define UBQP_WARP_VOLATILE 1
#endif
__device__ __forceinline__ int dp2a_lo(uint32_t a, uint32_t b, int c) {
    int d;
#if UBQP_WARP_VOLATILE
    asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
#else
    asm("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
#endif
    return d;
}
__device__ __forceinline__ int dp2a_hi(uint32_t a, uint32_t b, int c) {
    int d;
#if UBQP_WARP_VOLATILE
    asm volatile("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
#else
    asm("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
#endif
    return d;
}
__device__ __forceinline__ int max3i(int a, int b, int c) { return max(a, max(b, c)); }
__device__ __forceinline__ int min3i(int a, int b, int c) { return min(a, min(b, c)); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// K[li >> 4][li & 15] += v for a warp-UNIFORM local index li (v = 0 on every lane but the
// owner of k*), keeping every key in its register across the dispatch.
//   UBQP_WARP_DISPATCH 0 (default): one switch over li whose leaves are single in-place adds;
//   UBQP_WARP_DISPATCH 1: a switch over the chunk, then 16 predicated adds (measured the same
//   at n = 7000, slower at n <= 2500).
#ifndef UBQP_WARP_DISPATCH
#define UBQP_WARP_DISPATCH 0
#endif
template <int NCH>
__device__ __forceinline__ void add_key(int (&K)[NCH][16], int li, int v) {
#if UBQP_WARP_DISPATCH == 0
#define UBQP_W_A(C, E)                                                              \
    case 16 * C + E:                                                                \
        if constexpr (C < NCH) asm volatile("add.s32 %0, %0, %1;" : "+r"(K[C][E]) : "r"(v)); \
        break;
#define UBQP_W_C(C)                                                                         \
    UBQP_W_A(C, 0) UBQP_W_A(C, 1) UBQP_W_A(C, 2) UBQP_W_A(C, 3) UBQP_W_A(C, 4) UBQP_W_A(C, 5)     \
    UBQP_W_A(C, 6) UBQP_W_A(C, 7) UBQP_W_A(C, 8) UBQP_W_A(C, 9) UBQP_W_A(C, 10) UBQP_W_A(C, 11)   \
    UBQP_W_A(C, 12) UBQP_W_A(C, 13) UBQP_W_A(C, 14) UBQP_W_A(C, 15)
    switch (li) {
        UBQP_W_C(0) UBQP_W_C(1) UBQP_W_C(2) UBQP_W_C(3) UBQP_W_C(4) UBQP_W_C(5) UBQP_W_C(6)
        UBQP_W_C(7) UBQP_W_C(8) UBQP_W_C(9) UBQP_W_C(10) UBQP_W_C(11) UBQP_W_C(12) UBQP_W_C(13)
        default: break;
    }
#undef UBQP_W_C
#undef UBQP_W_A
#else
    const int e = li & 15;
#define UBQP_W_C(C)                                                                              \
    case C:                                                                                      \
        if constexpr (C < NCH) {                                                                 \
            _Pragma("unroll") for (int q = 0; q < 16; ++q)                                       \
                asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, %2;\n\t@p add.s32 %0, %0, %3;\n\t}" \
                             : "+r"(K[C][q]) : "r"(e), "r"(q), "r"(v));                           \
        }                                                                                        \
        break;
    switch (li >> 4) {
        UBQP_W_C(0) UBQP_W_C(1) UBQP_W_C(2) UBQP_W_C(3) UBQP_W_C(4) UBQP_W_C(5) UBQP_W_C(6)
        UBQP_W_C(7) UBQP_W_C(8) UBQP_W_C(9) UBQP_W_C(10) UBQP_W_C(11) UBQP_W_C(12) UBQP_W_C(13)
        default: break;
    }
#undef UBQP_W_C
#endif
}

}  // namespace
}  // namespace ubqp
