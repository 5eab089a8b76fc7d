// Microbenchmarks for the design of the sweep kernel (development aid, not product):
//   fp64 DFMA throughput, L2-resident read bandwidth, HBM read bandwidth,
//   L2-resident gather-style bandwidth (8-byte coalesced loads), DSMEM read bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_dfma(double *out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <int VEC>
__global__ void k_read(const double *__restrict__ in, size_t n, int passes, double *out) {
    double s = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x * VEC;
    for (int p = 0; p < passes; p++) {
        for (size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * VEC; i < n; i += stride) {
            if (VEC == 2) {
                double2 v = *reinterpret_cast<const double2 *>(in + i);
                s += v.x + v.y;
            } else {
                s += in[i];
            }
        }
    }
    if (s == 1.2345) out[0] = s;
}

// DSMEM: each CTA of a cluster of 2 reads its partner's shared memory
__global__ void __cluster_dims__(2, 1, 1) k_dsmem(double *out, int iters) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const double *peer = cl.map_shared_rank(buf, cl.block_rank() ^ 1);
    double s = 0;
    for (int it = 0; it < iters; it++)
        for (int i = threadIdx.x; i < 4096; i += blockDim.x) s += peer[i ^ (it & 31)];
    cl.sync();
    if (s == 1.2345) out[0] = s;
}
__global__ void k_lsmem(double *out, int iters) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    __syncthreads();
    double s = 0;
    for (int it = 0; it < iters; it++)
        for (int i = threadIdx.x; i < 4096; i += blockDim.x) s += buf[i ^ (it & 31)];
    if (s == 1.2345) out[0] = s;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    cudaMalloc(&out, sizeof(double) * 1 << 22);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    {   // DFMA
        int blocks = nsm * 8, thr = 256, iters = 4096;
        k_dfma<<<blocks, thr>>>(out, 16);
        cudaEventRecord(e0);
        k_dfma<<<blocks, thr>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 64 * iters * (double)blocks * thr;
        printf("DFMA: %.2f TFLOP/s fp64 (%.1f DFMA/clk/SM at 1965 MHz)\n", fl / ms / 1e9, fl / 2 / (ms * 1e-3) / nsm / 1.965e9);
    }
    for (size_t mb : {32, 64, 96, 4096}) {
        size_t n = mb * (1 << 20) / 8;
        double *in;
        cudaMalloc(&in, n * 8);
        cudaMemset(in, 0, n * 8);
        int passes = mb <= 96 ? 20 : 2;
        for (int vec : {1, 2}) {
            auto run = [&]() {
                if (vec == 1) k_read<1><<<nsm * 8, 512>>>(in, n, passes, out);
                else k_read<2><<<nsm * 8, 512>>>(in, n, passes, out);
            };
            run();
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("read %5zu MB x %d passes, %d-wide: %.0f GB/s\n", mb, passes, vec * 8, (double)n * 8 * passes / ms / 1e6);
        }
        cudaFree(in);
    }
    {
        int iters = 2000;
        k_dsmem<<<nsm, 512>>>(out, 10);
        cudaEventRecord(e0);
        k_dsmem<<<nsm, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("DSMEM read (cluster 2): %.0f GB/s total, %.1f B/clk/SM\n", 4096.0 * 8 * iters * nsm / ms / 1e6,
               4096.0 * 8 * iters / (ms * 1e-3) / 1.965e9);
        k_lsmem<<<nsm, 512>>>(out, 10);
        cudaEventRecord(e0);
        k_lsmem<<<nsm, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("local smem read: %.0f GB/s total, %.1f B/clk/SM\n", 4096.0 * 8 * iters * nsm / ms / 1e6,
               4096.0 * 8 * iters / (ms * 1e-3) / 1.965e9);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
