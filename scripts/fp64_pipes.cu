// fp64_pipes.cu -- measure B200 FP64 throughput: DFMA (FP64 ALU), DMMA
// (mma.sync.aligned.m8n8k4.f64, the legacy FP64 tensor path) and both mixed in
// one kernel.  Decides whether the FP64-bound DoGIP variants can use the
// tensor path as extra throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
            x4 = fma(x4, a, 1e-9); x5 = fma(x5, a, 1e-9); x6 = fma(x6, a, 1e-9); x7 = fma(x7, a, 1e-9);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a) {
    double c[8][2];
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3;
    const double b = a * 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mixed_kernel(double* out, int iters, double a, int dfma_per_dmma) {
    double c[4][2];
    for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-3;
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    const double b = a * 0.5;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(c[k][0], c[k][1], a, b);
        for (int r = 0; r < dfma_per_dmma; ++r) {
            x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
            x4 = fma(x4, a, 1e-9); x5 = fma(x5, a, 1e-9); x6 = fma(x6, a, 1e-9); x7 = fma(x7, a, 1e-9);
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, blocks = nsm * 4, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // DFMA: 64 fma per iteration per thread
    dfma_kernel<<<blocks, threads>>>(out, 16, 0.999);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma_flops = 2.0 * 64 * iters * (double)threads * blocks;
    printf("{\"dfma_tflops\": %.2f, ", dfma_flops / ms / 1e9);
    // DMMA m8n8k4: 2*8*8*4 = 512 flops per warp-instruction, 8 per iteration
    dmma_kernel<<<blocks, threads>>>(out, 16, 0.999);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmma_flops = 512.0 * 8 * iters * (double)(threads / 32) * blocks;
    printf("\"dmma_tflops\": %.2f, ", dmma_flops / ms / 1e9);
    // mixed: 4 DMMA (2048 flops/warp) + R x 8 DFMA per thread per iteration
    for (int R : {1, 2, 4, 8}) {
        mixed_kernel<<<blocks, threads>>>(out, 16, 0.999, R);
        cudaEventRecord(e0);
        mixed_kernel<<<blocks, threads>>>(out, iters, 0.999, R);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = (512.0 * 4 * (threads / 32) + 2.0 * 8 * R * threads) * iters * (double)blocks;
        const double t_dmma_alone = 512.0 * 4 * (threads / 32) * iters * (double)blocks / (dmma_flops / 1e3);
        printf("\"mixed_R%d_tflops\": %.2f, ", R, fl / ms / 1e9);
        (void)t_dmma_alone;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("\"sms\": %d, \"clock_khz_attr\": %d}\n", nsm, clk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
