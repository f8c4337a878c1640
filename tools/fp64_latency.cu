// FP64 pipe microbenchmark (why the two-sweep pass is latency-bound).
//   latency    one warp, one dependent chain of DFMA (or rcp.approx.ftz.f64 seeds): cycles per op
//   throughput one CTA per SM, W warps per SM-sub-partition, 8 independent DFMA chains per
//              thread: cycles per warp-instruction per SMSP
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_latency tools/fp64_latency.cu
// Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;  // dependent ops per chain

__global__ void k_lat_fma(double *out, long long *cyc, double a, double b) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_lat_rcp(double *out, long long *cyc) {
    double x = 1.5 + threadIdx.x * 1e-3;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) {
        double r;
        asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
        x = r;  // rcp(rcp(x)) ~ x: stays in range
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_thr_fma(double *out, long long *cyc, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N / 8; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h[1024];
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&out, 1 << 22);
    cudaMalloc(&cyc, 1024 * sizeof(long long));
    const double a = 0.999999, b = 1e-7;
    k_lat_fma<<<1, 32>>>(out, cyc, a, b);  // warm-up
    k_lat_fma<<<1, 32>>>(out, cyc, a, b);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    const double lat_fma = (double)h[0] / N;
    k_lat_rcp<<<1, 32>>>(out, cyc);
    k_lat_rcp<<<1, 32>>>(out, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    const double lat_rcp = (double)h[0] / N;
    printf("{\"sm\": %d, \"dfma_latency_cycles\": %.2f, \"rcp_approx_f64_latency_cycles\": %.2f, \"dfma_throughput\": [",
           nsm, lat_fma, lat_rcp);
    for (int w = 1; w <= 8; w *= 2) {  // warps per SMSP
        const int threads = 4 * 32 * w;
        k_thr_fma<<<nsm, threads>>>(out, cyc, a, b);
        k_thr_fma<<<nsm, threads>>>(out, cyc, a, b);
        cudaMemcpy(h, cyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int s = 0; s < nsm; ++s) mx = h[s] > mx ? h[s] : mx;
        const double warp_instr_per_smsp = (double)w * N * 8;  // per SMSP: w warps x 8N DFMA each
        printf("%s{\"warps_per_smsp\": %d, \"cycles_per_dfma_warp_instr_per_smsp\": %.3f}", w > 1 ? ", " : "", w,
               (double)mx / warp_instr_per_smsp);
    }
    printf("], \"error\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
