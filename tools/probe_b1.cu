// Microbenchmark: throughput of the legacy binary tensor-core MMA
// (mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc) on sm_100a,
// and a small exactness check against popc(a & b) on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_b1 probe_b1.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_b1(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CHAINS>
__global__ void k_tput(int iters, int *out, uint32_t seed) {
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = seed * (threadIdx.x + 7 * i + 1);
    for (int i = 0; i < 2; ++i) b[i] = seed ^ (threadIdx.x * 2654435761u + i);
    int d[CHAINS][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) mma_b1(d[c], a, b);
    }
    int s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 0x7fffffff) out[0] = s;
}

// one m16n8k256 product: A 16x256 bits (row), B 256x8 bits (col), fragments
// loaded from global in the documented layout
__global__ void k_one(const uint32_t *A, const uint32_t *B, int *D) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    uint32_t a[4], b[2];
    // A: a0 (row g, k 32t..32t+31) a1 (row g+8, same k) a2 (row g, k 128+32t..) a3 (row g+8, k 128+..)
    a[0] = A[g * 8 + t];
    a[1] = A[(g + 8) * 8 + t];
    a[2] = A[g * 8 + 4 + t];
    a[3] = A[(g + 8) * 8 + 4 + t];
    // B (col-major, column n = g): b0 k 32t.., b1 k 128+32t..
    b[0] = B[g * 8 + t];
    b[1] = B[g * 8 + 4 + t];
    int d[4] = {0, 0, 0, 0};
    mma_b1(d, a, b);
    // D: d0 (row g, col 2t) d1 (row g, col 2t+1) d2 (row g+8, col 2t) d3 (row g+8, 2t+1)
    D[g * 8 + 2 * t] = d[0];
    D[g * 8 + 2 * t + 1] = d[1];
    D[(g + 8) * 8 + 2 * t] = d[2];
    D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int *out;
    cudaMalloc(&out, 64);
    // exactness
    std::vector<uint32_t> A(16 * 8), B(8 * 8);
    srand(1);
    for (auto &x : A) x = (uint32_t)rand() * 2654435761u ^ rand();
    for (auto &x : B) x = (uint32_t)rand() * 2246822519u ^ rand();
    uint32_t *dA, *dB;
    int *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, 16 * 8 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    k_one<<<1, 32>>>(dA, dB, dD);
    std::vector<int> D(128);
    cudaError_t e = cudaMemcpy(D.data(), dD, 512, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
        return 1;
    }
    int bad = 0;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            int s = 0;
            for (int w = 0; w < 8; ++w) s += __builtin_popcount(A[r * 8 + w] & B[c * 8 + w]);
            if (s != D[r * 8 + c]) ++bad;
        }
    printf("{\"exact_mismatches\": %d", bad);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        dim3 grid(sms * 4), block(32 * warps);
        k_tput<8><<<grid, block>>>(16, out, 3);
        cudaEventRecord(e0);
        k_tput<8><<<grid, block>>>(iters, out, 3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double macs = (double)grid.x * warps * iters * 8 * (16.0 * 8 * 256);
        printf(", \"w%d_ms\": %.3f, \"w%d_Tbitmac_s\": %.1f", warps, ms, warps, macs / ms / 1e9);
    }
    printf("}\n");
    e = cudaGetLastError();
    if (e != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
