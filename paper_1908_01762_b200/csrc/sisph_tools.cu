// sisph_tools.cu — measurement helpers for bench.py (not on the hot path):
// the FP32 ALU roof that SURVEY.md §8(d) M3(b)/(c) divides by.  MEASURED_PEAKS.json
// carries HBM bandwidth and dense bf16 tensor throughput only; the pair passes
// and the neighbour build are issue-bound on FP32 / integer instructions, so
// their roofline needs the issue rate of this GPU at its current clocks.
//
//   sisph_tools_alu_peak(device, out[4]):
//     out[0]  FFMA   warp-instructions / s  (x 32 = lane FMAs / s; x 64 = FP32 flop/s)
//     out[1]  MUFU.RSQ warp-instructions / s
//     out[2]  the warp-instruction issue roof (= the FFMA rate: on sm_100 the FP32 pipe takes
//             one warp-instruction per scheduler per cycle, the issue limit itself)
//     out[3]  SM clock in MHz during the FFMA run (block 0's clock64 cycles over its own
//             %globaltimer span)
// Each kernel runs 8 independent dependency chains per thread (enough ILP to
// hide the 4-cycle FMA latency at 4 warps per scheduler) over a grid of
// 8 x SM-count blocks of 256 threads, and is timed with CUDA events after a
// warm-up launch.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int CHAINS = 8;

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_ffma(float* out, int iters, float a, float b, long long* cyc)
{
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = threadIdx.x * 1e-3f + c;
    const unsigned long long g0 = gtimer();
    const long long t0 = clock64();
    for (int k = 0; k < iters; k++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int c = 0; c < CHAINS; c++) x[c] = fmaf(x[c], a, b);
        }
    }
    const long long t1 = clock64();
    const unsigned long long g1 = gtimer();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.678f) out[0] = s;   // keep the chains live
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = (long long)(g1 - g0);   // ns
    }
}

__global__ void k_mufu(float* out, int iters)
{
    float x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; c++) x[c] = 1.0f + threadIdx.x * 1e-3f + c;
    for (int k = 0; k < iters; k++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
#pragma unroll
            for (int c = 0; c < CHAINS; c++) {
                float r;
                asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[c]));
                x[c] = r;
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHAINS; c++) s += x[c];
    if (s == 12345.678f) out[0] = s;
}

}  // namespace

extern "C" int sisph_tools_alu_peak(int device, double* out)
{
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = 8 * sms, threads = 256, iters = 4096;
    float* f = nullptr;
    long long* cyc = nullptr;
    if (cudaMalloc(&f, 64) != cudaSuccess || cudaMalloc(&cyc, 2 * sizeof(long long)) != cudaSuccess) return 2;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double warps = (double)blocks * threads / 32.0;
    const double per_warp = (double)iters * 16 * CHAINS;   // instructions of the measured op per warp
    float ms = 0;
    // FFMA
    k_ffma<<<blocks, threads>>>(f, iters, 0.999f, 1e-3f, cyc);
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(f, iters, 0.999f, 1e-3f, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[2] = {0, 0};
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    out[0] = warps * per_warp / (ms * 1e-3);
    out[3] = c[1] > 0 ? (double)c[0] / (double)c[1] * 1e3 : 0.0;   // cycles per ns x 1000 = MHz
    // MUFU
    k_mufu<<<blocks, threads>>>(f, iters / 4);
    cudaEventRecord(e0);
    k_mufu<<<blocks, threads>>>(f, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    out[1] = warps * per_warp / 4 / (ms * 1e-3);
    out[2] = out[0];   // issue roof: FP32 FFMA issues at one warp-instruction per scheduler per cycle
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(f);
    cudaFree(cyc);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
