// FP32 issue rates on one B200 SM, for the GEMM's GELU epilogue: scalar FFMA
// vs packed FFMA2 (fma.rn.f32x2) vs MUFU (ex2 / rcp), 8 independent chains per
// thread, 8 warps per SM (the epilogue's shape) and 32 warps per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a ffma2_probe.cu -o ffma2_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int kOp>
__global__ void probe(float* out, int iters, float s) {
  float a[8];
  uint64_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 1e-3f + i;
    const float lo = a[i], hi = a[i] + 0.5f;
    p[i] = (static_cast<uint64_t>(__float_as_uint(hi)) << 32) | __float_as_uint(lo);
  }
  const uint64_t m = (static_cast<uint64_t>(__float_as_uint(s)) << 32) | __float_as_uint(s);
  const uint64_t c = (static_cast<uint64_t>(__float_as_uint(0.25f)) << 32) | __float_as_uint(0.25f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (kOp == 0) a[i] = fmaf(a[i], s, 0.25f);
      if constexpr (kOp == 1) p[i] = ffma2(p[i], m, c);
      if constexpr (kOp == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if constexpr (kOp == 3) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += a[i] + __uint_as_float(static_cast<uint32_t>(p[i]));
  if (acc == 1234.5f) *out = acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  const char* names[] = {"ffma", "ffma2", "mufu_ex2", "mufu_rcp"};
  for (int warps : {8, 32}) {
    for (int op = 0; op < 4; ++op) {
      auto run = [&] {
        if (op == 0) probe<0><<<sms, 32 * warps>>>(o, iters, 0.999f);
        if (op == 1) probe<1><<<sms, 32 * warps>>>(o, iters, 0.999f);
        if (op == 2) probe<2><<<sms, 32 * warps>>>(o, iters, 0.999f);
        if (op == 3) probe<3><<<sms, 32 * warps>>>(o, iters, 0.999f);
      };
      run();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int clk_khz;
      cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
      // warp-instructions per SM per clock (at the reported max clock)
      const double instr = 5.0 * warps * iters * 8.0;
      const double clocks = ms * 1e-3 * clk_khz * 1e3;
      const double per_clk = instr / clocks;
      const double elems = per_clk * 32 * (op == 1 ? 2 : 1);
      std::printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"warp_instr_per_sm_clk\": %.3f, "
                  "\"lane_results_per_sm_clk\": %.1f}\n", names[op], warps, per_clk, elems);
    }
  }
  return 0;
}
