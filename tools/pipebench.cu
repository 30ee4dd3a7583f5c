// pipebench.cu — issue rates of the ascent's inner-loop instructions on this GPU (warp
// instructions per cycle per SM at 32 warps per SM), so the ascent roofline rests on measured
// pipe rates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipebench tools/pipebench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s\n", cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ int idp(uint32_t a, uint32_t b, int c) {
    int d;
    asm volatile("dp2a.lo.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ int vmax(int a, int b) {
    int d;
    asm volatile("max.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

// KIND 0: 16 IDP.2A per iteration (16 independent chains)
// KIND 2: the ascent's mix: 16 IDP.2A + 16 VIMNMX3 per iteration
// KIND 3: 16 IMAD per iteration
// KIND 4: 16 IDP.2A + 16 two-input IMNMX;  KIND 5: 16 IDP.2A + 16 LOP3;  KIND 6: 16 IDP.2A with
// the ascent's operand sharing (one multiplier register, one row word per 4) + 16 VIMNMX3 whose
// two data operands are the IDP results just produced (max and min over the same pair);
// KIND 7: 16 IDP.2A + 32 two-input IMNMX (the argmax without 3-input min/max)
__device__ __forceinline__ int idph(uint32_t a, uint32_t b, int c) {
    int d;
    asm volatile("dp2a.hi.s32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// KIND 9: the warp ascent's loop, per 32-bit row word: 4 IDP.2A (vector multipliers (C,0) and
// (0,C), the word shared) into 4 keys, then a 3-input max and a 3-input min over each key pair
template <int KIND>
__global__ void bench(int *out, uint32_t a, uint32_t b, int iters) {
    if (KIND == 11 || KIND == 12 || KIND == 13) {
        // the replica with the row words read from shared memory, one LDS.128 per 4 words, like
        // the kernel (KIND 12: each chunk's load address depends on the max chain two chunks back
        // through a runtime zero, to force IDP.2A / VIMNMX3 interleaving)
        __shared__ uint4 srow[14 * 32];
        for (int i = threadIdx.x; i < 14 * 32; i += blockDim.x) srow[i] = make_uint4(a * i, b ^ i, a + i, b - i);
        __syncthreads();
        const int lane = threadIdx.x & 31;
        int K[224];
#pragma unroll
        for (int i = 0; i < 224; ++i) K[i] = threadIdx.x * (i + 3);
        uint32_t a0 = KIND == 13 ? a & 0xFFFFu : a * threadIdx.x & 0xFFFFu;   // 13: warp-uniform multipliers
        uint32_t a1 = KIND == 13 ? a << 16 : (a * threadIdx.x) << 16;
        int m0 = 0, m1 = 0, n0 = 0, n1 = 0;
        const uint32_t zero = b >> 31;                    // 0 at run time, unknown to the compiler
        for (int it = 0; it < iters; ++it) {
            int hist[14];
#pragma unroll
            for (int c = 0; c < 14; ++c) {
                uint32_t addr = static_cast<uint32_t>(__cvta_generic_to_shared(&srow[32 * c + lane]));
                if (KIND == 12 && c >= 2)
                    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(addr) : "r"(hist[c - 2]), "r"(zero), "r"(addr));
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    int &k0 = K[16 * c + 4 * q], &k1 = K[16 * c + 4 * q + 1], &k2 = K[16 * c + 4 * q + 2],
                        &k3 = K[16 * c + 4 * q + 3];
                    k0 = idp(a0, wv[q], k0);
                    k1 = idp(a1, wv[q], k1);
                    k2 = idph(a0, wv[q], k2);
                    k3 = idph(a1, wv[q], k3);
                    m0 = max(m0, max(k0, k1));
                    n0 = min(n0, min(k0, k1));
                    m1 = max(m1, max(k2, k3));
                    n1 = min(n1, min(k2, k3));
                }
                hist[c] = m0;
            }
            a0 ^= static_cast<uint32_t>(m0 & 1);
        }
        int s = m0 ^ m1 ^ n0 ^ n1;
#pragma unroll
        for (int i = 0; i < 224; ++i) s ^= K[i];
        if (s == 0x12345) out[threadIdx.x] = s;
        return;
    }
    if (KIND == 9 || KIND == 10) {
        constexpr int NWD = KIND == 9 ? 8 : 56;           // row words per step (4 keys each)
        int K[4 * NWD];
#pragma unroll
        for (int i = 0; i < 4 * NWD; ++i) K[i] = threadIdx.x * (i + 3);
        uint32_t a0 = a * threadIdx.x & 0xFFFFu, a1 = (a * threadIdx.x) << 16;
        uint32_t w = b ^ threadIdx.x;
        int m0 = 0, m1 = 0, n0 = 0, n1 = 0;
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int q = 0; q < NWD; ++q) {
                const uint32_t ww = w + q;
                int &k0 = K[4 * q], &k1 = K[4 * q + 1], &k2 = K[4 * q + 2], &k3 = K[4 * q + 3];
                k0 = idp(a0, ww, k0);
                k1 = idp(a1, ww, k1);
                k2 = idph(a0, ww, k2);
                k3 = idph(a1, ww, k3);
                m0 = max(m0, max(k0, k1));
                n0 = min(n0, min(k0, k1));
                m1 = max(m1, max(k2, k3));
                n1 = min(n1, min(k2, k3));
            }
            w = w * 1664525u + static_cast<uint32_t>(m0 ^ n1);
        }
        int s = m0 ^ m1 ^ n0 ^ n1;
#pragma unroll
        for (int i = 0; i < 4 * NWD; ++i) s ^= K[i];
        if (s == 0x12345) out[threadIdx.x] = s;
        return;
    }
    int k[16], m[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { k[i] = threadIdx.x * (i + 1); m[i] = threadIdx.x ^ i; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (KIND == 0 || KIND == 2) k[i] = idp(a, b + i, k[i]);
            if (KIND == 3) k[i] = k[i] * static_cast<int>(a) + static_cast<int>(b);
            if (KIND == 2) m[i] = (i & 1) ? min(m[i], min(k[i], k[i ^ 1])) : max(m[i], max(k[i], k[i ^ 1]));
            if (KIND == 4) { k[i] = idp(a, b + i, k[i]); m[i] = max(m[i], k[i]); }
            if (KIND == 5) { k[i] = idp(a, b + i, k[i]); m[i] = m[i] ^ (k[i] & 0x5555); }
            if (KIND == 6) k[i] = idp((i & 1) ? a : b, b + (i >> 2), k[i]);
            if (KIND == 1) m[i] = vmax(vmax(m[i], m[(i + 5) & 15]), m[(i + 9) & 15]);
            if (KIND == 8) m[i] = vmax(m[i], m[(i + 5) & 15]);
            if (KIND == 7) { k[i] = idp(a, b + i, k[i]); m[i] = max(m[i], k[i]); m[i ^ 1] = min(m[i ^ 1], k[i]); }

        }
        if (KIND == 6) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                m[i] = max(m[i], max(k[i], k[i + 1]));
                m[i + 1] = min(m[i + 1], min(k[i], k[i + 1]));
                m[i + 2] = max(m[i + 2], max(k[i + 2], k[i + 3]));
                m[i + 3] = min(m[i + 3], min(k[i + 2], k[i + 3]));
            }
        }
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s ^= k[i] ^ m[i];
    if (s == 0x12345) out[threadIdx.x] = s;
}

int main() {
    int *out;
    CK(cudaMalloc(&out, 4096));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 8192, threads = 1024, blocks = sms;   // 32 warps per SM
    const char *names[] = {"IDP.2A", "VIMNMX3 alone", "IDP.2A + VIMNMX3 (1:1)", "IMAD", "IDP.2A + IMNMX (1:1)",
                           "IDP.2A + LOP3 (1:1)", "IDP.2A + VIMNMX3 (1:1/4)", "IDP.2A + 2 IMNMX (1:2)", "IMNMX alone",
                           "ascent loop (per word 4 IDP + 4 VIMNMX3)"};
    const int ops[] = {16, 16, 32, 16, 32, 32, 32, 48, 16, 64};
    for (int kind = 0; kind < 10; ++kind) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) bench<0><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 1) bench<1><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 8) bench<8><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 9) bench<9><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 2) bench<2><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 3) bench<3><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 4) bench<4><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 5) bench<5><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 6) bench<6><<<blocks, threads>>>(out, 3, 5, iters);
            if (kind == 7) bench<7><<<blocks, threads>>>(out, 3, 5, iters);

            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double warp_ops = static_cast<double>(blocks) * (threads / 32) * iters * ops[kind];
        const double ghz = 1.965;                              // SM clock under load (bench clocks)
        printf("%-24s %8.3f ms  %.3f warp-instr/cycle/SM  (%.2f lanes/cycle/SMSP) @%.3f GHz\n", names[kind], best,
               warp_ops / (best * 1e-3 * ghz * 1e9) / sms, warp_ops * 32 / (best * 1e-3 * ghz * 1e9) / sms / 4, ghz);
    }
    // the loop replica at the warp kernel's occupancy and beyond; 224 keys per lane like n = 7000
    for (int wps : {8}) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            bench<10><<<sms, 32 * wps>>>(out, 3, 5, iters / 7);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double warp_ops = static_cast<double>(sms) * wps * (iters / 7) * 56 * 8;
        printf("ascent loop replica, 224 keys, %2d warps/SM: %.3f warp-instr/cycle/SM = %.1f variable updates/SM cycle\n",
               wps, warp_ops / (best * 1e-3 * 1.965e9) / sms, warp_ops / (best * 1e-3 * 1.965e9) / sms * 16);
    }
    for (int kind : {11, 12, 13}) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (kind == 11) bench<11><<<sms, 32 * 8>>>(out, 3, 5, iters / 7);
            else if (kind == 12) bench<12><<<sms, 32 * 8>>>(out, 3, 5, iters / 7);
            else bench<13><<<sms, 32 * 8>>>(out, 3, 5, iters / 7);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double warp_ops = static_cast<double>(sms) * 8 * (iters / 7) * 56 * 8;
        printf("replica with LDS row words%s, 8 warps/SM: %.1f variable updates/SM cycle\n",
               kind == 12 ? " + lag-2 address token" : (kind == 13 ? ", warp-uniform multipliers" : ""),
               warp_ops / (best * 1e-3 * 1.965e9) / sms * 16);
    }
    for (int wps : {4, 8, 12, 16, 24}) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            bench<9><<<sms, 32 * wps>>>(out, 3, 5, iters);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double warp_ops = static_cast<double>(sms) * wps * iters * 64;
        printf("ascent loop replica, %2d warps/SM: %.3f warp-instr/cycle/SM = %.1f variable updates/SM cycle\n", wps,
               warp_ops / (best * 1e-3 * 1.965e9) / sms, warp_ops / (best * 1e-3 * 1.965e9) / sms * 16);
    }
    return 0;
}
