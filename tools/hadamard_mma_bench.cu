// Experiment (VERDICT r1 item 4 / north_star: "tensor cores only if a
// Hadamard-block MMA formulation measurably beats the shuffle butterfly"):
// throughput of the 32-point fp64 Hadamard row transform of the large-path
// row stage (hadamard_reg<5>: 5 x 16 butterflies in registers, one row per
// thread) against a DMMA formulation on the fp64 tensor cores
// (mma.sync.m8n8k4.f64): a warp transforms 32 rows as 4 tiles of 8 rows;
// per tile and 8-column group, Z_g H_8 = two k = 4 DMMAs, then H_4 across
// the 4 groups as register butterflies (H_32 = H_4 (x) H_8).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hmb tools/hadamard_mma_bench.cu && /tmp/hmb
#include <cuda_runtime.h>

#include <cstdio>

constexpr int ITERS = 2000;

__device__ __forceinline__ void had32(double* x) {
#pragma unroll
    for (int hb = 0; hb < 5; ++hb) {
        const int h = 1 << hb;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if ((i & h) == 0) {
                const double a = x[i], b = x[i + h];
                x[i] = a + b;
                x[i + h] = a - b;
            }
    }
}

__global__ void k_reg(double* out) {
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = (threadIdx.x + i) * 1e-3;
    for (int it = 0; it < ITERS; ++it) {
        had32(x);
        if ((it & 7) == 7) {
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] *= 0x1p-20;  // keep the values finite (H H = 32 I)
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__global__ void k_mma(double* out) {
    const int lane = threadIdx.x & 31;
    // B fragments of H_8 (scaled by 1/32 so the iteration stays finite): element (k, n),
    // k = lane % 4 (+4 for the second k-chunk), n = lane / 4
    const int k0 = lane & 3, n0 = lane >> 2;
    const double b0 = (__popc(k0 & n0) & 1 ? -1.0 : 1.0) * 0.03125;
    const double b1 = (__popc((k0 + 4) & n0) & 1 ? -1.0 : 1.0) * 0.03125;
    // 4 row tiles x 4 column groups x 2 A values per lane = the same 32 doubles per thread
    double a[4][4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            a[t][g][0] = (lane + t + g) * 1e-3;
            a[t][g][1] = (lane - t + g) * 1e-3;
        }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            double d[4][2];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                double e0, e1;
                dmma(e0, e1, a[t][g][0], b0, 0.0, 0.0);
                dmma(d[g][0], d[g][1], a[t][g][1], b1, e0, e1);
            }
            // H_4 across the groups (butterflies); D's columns feed the next A (a
            // fixed column permutation of the tile -- the same instruction count)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const double p0 = d[0][v] + d[1][v], p1 = d[0][v] - d[1][v];
                const double p2 = d[2][v] + d[3][v], p3 = d[2][v] - d[3][v];
                a[t][0][v] = p0 + p2;
                a[t][1][v] = p1 + p3;
                a[t][2][v] = p0 - p2;
                a[t][3][v] = p1 - p3;
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int g = 0; g < 4; ++g) s += a[t][g][0] + a[t][g][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * nsm * 8 * 256);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int occ : {2, 4, 8}) {
        const int grid = nsm * occ;
        float ms[2];
        for (int which = 0; which < 2; ++which) {
            for (int rep = 0; rep < 2; ++rep) {  // warm-up, then timed
                cudaEventRecord(a);
                if (which == 0) k_reg<<<grid, 256>>>(out);
                else k_mma<<<grid, 256>>>(out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                cudaEventElapsedTime(&ms[which], a, b);
            }
        }
        // 32-point transforms: every thread owns 32 rows' worth of data per iteration
        // (k_reg: 1 row per thread; k_mma: 32 rows per warp = 1 per thread)
        const double rows = double(grid) * 256 * ITERS;
        printf("CTAs/SM %d: butterfly %.3f ms (%.2f G rows/s)  dmma %.3f ms (%.2f G rows/s)  ratio %.2f\n", occ,
               ms[0], rows / ms[0] / 1e6, ms[1], rows / ms[1] / 1e6, ms[1] / ms[0]);
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    return 0;
}
