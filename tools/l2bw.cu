// l2bw.cu — what the ascent's row stream can get out of L2 ("the row bound").
//
// Every warp repeatedly picks a row of an L2-resident int8 matrix (Q-shaped: rows x ld bytes,
// 51 MB at 7000 x 7168) and reads the whole row, like one flip step of the ascent:
//   ldg:  each lane loads its 16-byte pieces with LDG.128 (the CTA kernel's path, through L1)
//   tma:  one bulk copy (cp.async.bulk) of the row into shared memory + mbarrier wait, then LDS
// The next row index depends on the data just read (dep = 1: one row in flight per warp, the
// ascent's dependent chain) or not (dep = 0: independent rows, pure bandwidth).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw tools/l2bw.cu && ./l2bw
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int DEP>
__global__ void ldg_rows(const uint8_t *__restrict__ Q, int rows, int ld, int row_bytes, int iters,
                         uint32_t *out) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0, r = (gw * 2654435761u) % rows;
    for (int it = 0; it < iters; ++it) {
        const uint4 *p = reinterpret_cast<const uint4 *>(Q + static_cast<size_t>(r) * ld);
        uint32_t x = 0;
#pragma unroll 4
        for (int o = lane; o < row_bytes / 16; o += 32) {
            const uint4 v = __ldg(p + o);
            x ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        acc += x;
        if (DEP) x = __reduce_xor_sync(0xFFFFFFFFu, x);
        r = (r * 1103515245u + 12345u + (DEP ? (x & 1u) : 0u)) % rows;
    }
    if (acc == 0x12345678u) out[gw] = acc;
}

template <int DEP>
__global__ void tma_rows(const uint8_t *__restrict__ Q, int rows, int ld, int row_bytes, int iters,
                         uint32_t *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t *buf = sm + w * (row_bytes + 128);
    uint64_t *bar = reinterpret_cast<uint64_t *>(buf + row_bytes);
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint32_t acc = 0, r = (gw * 2654435761u) % rows, phase = 0;
    for (int it = 0; it < iters; ++it) {
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                         "r"(row_bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(Q + static_cast<size_t>(r) * ld)),
                "r"(row_bytes), "r"(smem_u32(bar)) : "memory");
        }
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
        phase ^= 1;
        uint32_t x = 0;
        for (int o = lane; o < row_bytes / 16; o += 32) {
            const uint4 v = reinterpret_cast<const uint4 *>(buf)[o];
            x ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        acc += x;
        x = __reduce_xor_sync(0xFFFFFFFFu, x);     // also orders the reads before the next copy
        r = (r * 1103515245u + 12345u + (DEP ? (x & 1u) : 0u)) % rows;
    }
    if (acc == 0x12345678u) out[gw] = acc;
}

int main(int argc, char **argv) {
    const int rows = argc > 1 ? atoi(argv[1]) : 7000;
    const int ld = argc > 2 ? atoi(argv[2]) : 7168;
    const int row_bytes = argc > 3 ? atoi(argv[3]) : ld;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    uint8_t *Q;
    uint32_t *out;
    CK(cudaMalloc(&Q, static_cast<size_t>(rows) * ld));
    CK(cudaMemset(Q, 1, static_cast<size_t>(rows) * ld));
    CK(cudaMalloc(&out, 1 << 24));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    printf("rows=%d ld=%d row_bytes=%d (%.1f MB) sms=%d\n", rows, ld, row_bytes, rows * (double)ld / 1e6, sms);
    const int iters = 2000;
    for (int kind = 0; kind < 4; ++kind) {
        const bool tma = kind >= 2;
        const int dep = kind & 1;
        for (int wpsm : {4, 8, 12, 16, 24, 32, 48}) {
            const int threads = 128;
            const int wpb = threads / 32;
            const int blocks = sms * wpsm / wpb;
            const size_t smem = tma ? static_cast<size_t>(wpb) * (row_bytes + 128) : 0;
            if (tma && smem * (wpsm / wpb) > 220 * 1024) continue;
            auto launch = [&]() {
                if (!tma) {
                    if (dep) ldg_rows<1><<<blocks, threads>>>(Q, rows, ld, row_bytes, iters, out);
                    else ldg_rows<0><<<blocks, threads>>>(Q, rows, ld, row_bytes, iters, out);
                } else {
                    if (dep) tma_rows<1><<<blocks, threads, smem>>>(Q, rows, ld, row_bytes, iters, out);
                    else tma_rows<0><<<blocks, threads, smem>>>(Q, rows, ld, row_bytes, iters, out);
                }
            };
            if (tma) {
                CK(cudaFuncSetAttribute(tma_rows<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                CK(cudaFuncSetAttribute(tma_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            }
            launch();
            CK(cudaGetLastError());
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double bytes = static_cast<double>(blocks) * wpb * iters * row_bytes;
            printf("%s dep=%d warps/SM=%2d: %8.3f ms  %7.2f TB/s  %6.1f B/clk/SM@1.965GHz  rows/s %.3g\n",
                   tma ? "tma" : "ldg", dep, wpsm, ms, bytes / ms / 1e9, bytes / ms / 1e-3 / sms / 1.965e9,
                   static_cast<double>(blocks) * wpb * iters / ms * 1e3);
        }
    }
    return 0;
}
