// fp64_latency.cu -- B200 DFMA throughput vs resident warps per SM and ILP
// (independent FMA chains per thread), with the coefficient as an immediate
// (like the generated DoGIP body) or a register.  Answers whether the apply
// kernel's ~50 % FP64 pipe utilisation is a latency (warps x ILP) limit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, bool IMM>
__global__ void chains(double* out, int iters, double a) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int k = 0; k < ILP; ++k) x[k] = IMM ? fma(x[k], 0.999755859375, 0.0078125) : fma(x[k], a, 0.0078125);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, bool IMM>
void run(double* out, int nsm, int clk_khz, int ctas_per_sm) {
    const int threads = 128;
    const int smem = (227 * 1024) / ctas_per_sm - 1024;
    auto k = chains<ILP, IMM>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2048;
    k<<<nsm * ctas_per_sm, threads, smem>>>(out, 8, 0.999);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<nsm * ctas_per_sm, threads, smem>>>(out, iters, 0.999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = (double)iters * 16 * ILP * threads * nsm * ctas_per_sm;
    const double lanes_per_clk = fmas / (ms * 1e-3) / nsm / (clk_khz * 1e3);
    printf("{\"warps_per_sm\": %d, \"ilp\": %d, \"imm\": %d, \"tflops\": %.2f, \"fma_lanes_per_clk_sm\": %.1f}\n",
           ctas_per_sm * 4, ILP, (int)IMM, 2 * fmas / ms / 1e9, lanes_per_clk);
}

int main() {
    int nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * 128 * nsm * 16);
    for (int c : {1, 2, 3, 4, 8}) {
        run<1, true>(out, nsm, clk, c);
        run<2, true>(out, nsm, clk, c);
        run<3, true>(out, nsm, clk, c);
        run<4, true>(out, nsm, clk, c);
        run<8, true>(out, nsm, clk, c);
        run<4, false>(out, nsm, clk, c);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
