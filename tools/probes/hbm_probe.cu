// HBM ceilings on one B200 for the roofline discussion: write-only (st.global.v4),
// read-only (ld.global.nc.v4 + reduction), and copy (1 read : 1 write) and
// 1 read : 8 writes (the simulated-mesh all-gather fan-out), 1 GiB working sets;
// and the strided gather ceiling: `run` bytes out of every `stride`-byte row
// into a contiguous output (what a conversion that shards the innermost dim
// reads: RRR->RRS012 of a [512,512,256] bf16 tensor takes 64 B of every
// 512 B row), as GB/s of bytes moved (read + written).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a hbm_probe.cu -o hbm_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void write_k(uint4* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, i, i, i);
}
__global__ void read_k(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}
__global__ void copy_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + i));
    d[i] = v;
  }
}
__global__ void fan8_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  // d holds 8 consecutive n-element destinations
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + i));
#pragma unroll
    for (int j = 0; j < 8; ++j) d[j * n + i] = v;
  }
}

__global__ void gather_k(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n,
                         unsigned run16, unsigned stride16) {
  // n output chunks; chunk i = row i / run16, column i % run16
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t row = i / run16, c = i - row * run16;
    uint4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + row * stride16 + c));
    d[i] = v;
  }
}

int main() {
  const size_t bytes = size_t(1) << 30, n = bytes / 16;
  uint4 *a, *b, *c; unsigned* o;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&c, bytes); cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto time = [&](auto f, int reps) { f(); cudaDeviceSynchronize(); cudaEventRecord(e0); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / reps; };
  for (int mult : {4, 8, 16}) {
    const int grid = sms * mult;
    float w = time([&] { write_k<<<grid, 256>>>(a, n); }, 20);
    float r = time([&] { read_k<<<grid, 256>>>(a, n, o); }, 20);
    float cp = time([&] { copy_k<<<grid, 256>>>(a, b, n); }, 20);
    const size_t nf = n / 8;  // 128 MiB source, 1 GiB of writes
    float f8 = time([&] { fan8_k<<<grid, 256>>>(a, c, nf); }, 20);
    printf("{\"grid_per_sm\": %d, \"write_only_gbs\": %.1f, \"read_only_gbs\": %.1f, \"copy_gbs\": %.1f, \"fanout8_gbs\": %.1f}\n",
           mult, bytes / w / 1e6, bytes / r / 1e6, 2.0 * bytes / cp / 1e6, 9.0 * (bytes / 8) / f8 / 1e6);
  }
  for (unsigned stride : {512u, 4096u}) {
    for (unsigned run : {32u, 64u, 128u, 256u, 512u}) {
      if (run > stride) continue;
      const size_t rows = bytes / stride, nout = rows * (run / 16);
      float best = 1e30f;
      for (int mult : {4, 8, 16}) {
        const int grid = sms * mult;
        float t = time([&] { gather_k<<<grid, 256>>>(a, b, nout, run / 16, stride / 16); }, 20);
        best = t < best ? t : best;
      }
      printf("{\"gather_stride\": %u, \"run\": %u, \"moved_bytes\": %zu, \"gbs\": %.1f}\n", stride, run,
             2 * nout * 16, 2.0 * nout * 16 / best / 1e6);
    }
  }
  return 0;
}
