// red_f64.cu -- B200 throughput of red.global.add.f64 (the apply kernel's scatter) vs
// plain stores, on an L2-resident / HBM-sized vector, with the apply's access shape
// (each warp touches a few contiguous runs) and with neighbouring lanes colliding.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_f64 red_f64.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>   // 0: red.add.f64, 1: st.global.f64, 2: red.add.f64 with 2 lanes per address
__global__ void scatter(double* y, long n, int per_thread, long stride_lane) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long nthreads = (long)gridDim.x * blockDim.x;
    for (int k = 0; k < per_thread; ++k) {
        long i = (t + k * nthreads);
        if (MODE == 2) i = (i >> 1);
        i = (i * stride_lane) % n;
        if (MODE == 1) y[i] = 1.0;
        else asm volatile("red.global.add.f64 [%0], %1;" ::"l"(y + i), "d"(1.0) : "memory");
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (long n : {1L << 23, 1L << 27}) {   // 64 MB (L2-resident), 1 GB
        double* y;
        cudaMalloc(&y, n * sizeof(double));
        cudaMemset(y, 0, n * sizeof(double));
        const int threads = 256, blocks = nsm * 8, per = 64;
        const double ops = (double)threads * blocks * per;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int mode = 0; mode < 3; ++mode)
            for (long stride : {1L, 3L}) {
                auto k = mode == 0 ? scatter<0> : mode == 1 ? scatter<1> : scatter<2>;
                k<<<blocks, threads>>>(y, n, per, stride);
                cudaEventRecord(e0);
                for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(y, n, per, stride);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("{\"n_bytes\": %ld, \"mode\": \"%s\", \"lane_stride\": %ld, \"Gops_per_s\": %.1f}\n",
                       n * 8, mode == 0 ? "red.add.f64" : mode == 1 ? "st.f64" : "red.add.f64 2 lanes/addr", stride,
                       5 * ops / ms / 1e6);
            }
        cudaFree(y);
    }
    return 0;
}
