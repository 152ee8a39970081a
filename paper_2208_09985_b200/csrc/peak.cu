// Integer-ALU issue-rate microbenchmark (the roofline denominator of K1,
// P = N_SM * R_ALU * f_SM with R_ALU measured on the box).
// Eight independent LOP3 chains per thread; the ALU pipe (LOP3/SHF/IADD3) is
// the pipe K1's bitvector logic issues on.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/scrooge_b200.h"

namespace {

__global__ void __launch_bounds__(256) k_lop3_peak(unsigned* out, int iters, long long* cycles) {
    unsigned a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * (k + 3) + blockIdx.x;
    const unsigned b = out[0] | 0x0F0F0F0Fu, c = out[1] | 0x33333333u;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
    }
    __syncthreads();
    const long long t1 = clock64();
    unsigned s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= a[k];
    if (s == 0x9E3779B9u) out[2] = s;  // keep the chains alive
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

}  // namespace

static int alu_peak(int device, double* ops_per_clk_per_sm, double* sm_mhz, double* ops_per_s) {
    if (cudaSetDevice(device) != cudaSuccess) return SG_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    unsigned* out = nullptr;
    long long* cyc = nullptr;
    if (cudaMalloc(&out, 16) != cudaSuccess) return SG_CUDA;
    if (cudaMalloc(&cyc, sizeof(long long) * blocks) != cudaSuccess) return SG_CUDA;
    cudaMemset(out, 0, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_lop3_peak<<<blocks, threads>>>(out, iters / 8, cyc);  // warm-up
    cudaEventRecord(e0);
    k_lop3_peak<<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> c(static_cast<size_t>(blocks));
    cudaMemcpy(c.data(), cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
    const cudaError_t err = cudaGetLastError();
    cudaFree(out);
    cudaFree(cyc);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (err != cudaSuccess) return SG_CUDA;
    const long long maxc = *std::max_element(c.begin(), c.end());
    const double ops = static_cast<double>(blocks) * threads * iters * 32.0;
    if (ops_per_clk_per_sm) *ops_per_clk_per_sm = ops / (static_cast<double>(sms) * maxc);
    if (sm_mhz) *sm_mhz = maxc / (ms * 1e-3) / 1e6;
    if (ops_per_s) *ops_per_s = ops / (ms * 1e-3);
    return SG_OK;
}

extern "C" int sg_alu_peak(int device, double* ops_per_clk_per_sm, double* sm_mhz,
                           double* ops_per_s) {
    int prev = -1;  // the caller's current device is restored
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    const int rc = alu_peak(device, ops_per_clk_per_sm, sm_mhz, ops_per_s);
    if (prev >= 0) cudaSetDevice(prev);
    return rc;
}
