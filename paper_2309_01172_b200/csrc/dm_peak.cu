// dm_peak.cu — FP64 issue-rate microbenchmark used as the roofline
// denominator of the Mode B (generated-candidate) kernels: 8 independent
// DMUL+DADD chains per thread (no FMA: -fmad=false), a full grid of
// 8 CTAs x 256 threads per SM.  2 * 8 * iters fp64 ops per thread.
#include "dm_common.cuh"
#include "dm_abi_util.cuh"

namespace dm {
__global__ void __launch_bounds__(256) fp64_peak_kernel(int64_t iters, double* sink) {
    double a = 1.0 + 1e-16 * threadIdx.x, b = 1e-300;
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7;
    for (int64_t i = 0; i < iters; ++i) {
        x0 = __dadd_rn(__dmul_rn(x0, a), b); x1 = __dadd_rn(__dmul_rn(x1, a), b);
        x2 = __dadd_rn(__dmul_rn(x2, a), b); x3 = __dadd_rn(__dmul_rn(x3, a), b);
        x4 = __dadd_rn(__dmul_rn(x4, a), b); x5 = __dadd_rn(__dmul_rn(x5, a), b);
        x6 = __dadd_rn(__dmul_rn(x6, a), b); x7 = __dadd_rn(__dmul_rn(x7, a), b);
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 42.0) sink[0] = s;
}

// ALU-pipe issue rate: 8 independent LOP3 (3-input xor) chains per thread,
// a full grid of 8 CTAs x 256 threads per SM; the roofline denominator of
// the split sweep's inner loop (3 ALU-pipe instructions per candidate pair:
// FSEL + SEL + IADD3 halves), measured independently of that loop.
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__global__ void __launch_bounds__(256) alu_peak_kernel(int64_t iters, uint32_t* sink) {
    uint32_t k0 = threadIdx.x * 0x9E3779B9u, k1 = blockIdx.x ^ 0x85EBCA6Bu;
    uint32_t x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
             x7 = x0 + 7;
    for (int64_t i = 0; i < iters; ++i) {
        x0 = xor3(x0, k0, k1); x1 = xor3(x1, k0, k1); x2 = xor3(x2, k0, k1); x3 = xor3(x3, k0, k1);
        x4 = xor3(x4, k1, k0); x5 = xor3(x5, k1, k0); x6 = xor3(x6, k1, k0); x7 = xor3(x7, k1, k0);
    }
    uint32_t s = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
    if (s == 0x12345678u) sink[0] = s;
}
}  // namespace dm

extern "C" int dm_microbench_alu(int64_t iters, uint32_t* sink, int64_t* ops, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int grid = sms * 8;
    dm::alu_peak_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(iters, sink);
    DM_CHECK_LAUNCH();
    if (ops) *ops = (int64_t)grid * 256 * 8 * iters;
    return DM_OK;
}

extern "C" int dm_microbench_fp64(int64_t iters, double* sink, int64_t* ops, void* stream) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int grid = sms * 8;
    dm::fp64_peak_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(iters, sink);
    DM_CHECK_LAUNCH();
    if (ops) *ops = (int64_t)grid * 256 * 16 * iters;
    return DM_OK;
}
