// Dense bf16 GEMM on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
//   C[M,N] = epilogue( A[M,K] . Bt[N,K]^T ),  A, Bt bf16 K-contiguous
//   (Bt is the nn.Linear weight layout [out_features, in_features]),
//   fp32 accumulation in TMEM, output bf16 or fp32, optional exact-erf GELU.
//
// This is the local contraction of every sharded-matmul strategy of the
// reference catalog (proj/src/intraop.cpp:141-234): each device multiplies
// its shards; the strategy's layout conversions and partial-sum all-reduce
// run around it in the runtime.
//
// Two persistent, warp-specialized kernels (10 warps each):
//   warp 0       TMA producer: 64-wide K slabs of A and B into a kStages-
//                deep smem ring, 128B swizzle, mbarrier complete_tx;
//   warp 1       owns the TMEM allocation (2 accumulators, so the epilogue
//                of tile i overlaps the MMAs of tile i+1); lane 0 issues
//                tcgen05.mma and tcgen05.commit's each ring slot back;
//   warps 2..9   epilogue: tcgen05.ld 32x32b.x16 from TMEM (warp w reads
//                lanes 32*(w%4)..+31, half the columns each), GELU /
//                convert, 16-column stores.
// gemm_bf16_tcgen05       cta_group::1, 128 x BN tiles (BN 128 / 256);
// gemm_bf16_tcgen05_pair  cta_group::2 on a 2-CTA cluster, 256 x 256 tiles
//                         (each SM stages half of B: less smem fill per MMA).
// Both take a batch of problems in one launch and can fuse a reduction
// across problems (GemmArgs.reduce / .fan). Tails in M, N and K are handled
// by TMA zero fill plus masked stores.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <tuple>

namespace apl {

extern std::atomic<uint64_t> g_launches;

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128-byte swizzle row of bf16
constexpr int kEpiWarps = 8;  // 2 per TMEM lane quarter, each taking half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y)
      : "memory");
}

// Elected-lane forms for the whole-warp TMA producer (warp-uniform operands,
// one lane issues; see mma_bf16_elect).
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(smem_addr(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_e(void* dst, const CUtensorMap* map, uint64_t* bar,
                                              int x, int y) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(x), "r"(y)
      : "memory");
}

// K-major, 128B-swizzled operand tile: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t smem_desc(const void* tile) {
  const uint64_t addr = smem_addr(tile);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= uint64_t(1) << 16;                // leading byte offset (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;        // stride byte offset: 8 rows x 128 B
  d |= uint64_t(1) << 46;                // descriptor version (sm_100)
  d |= uint64_t(2) << 61;                // SWIZZLE_128B
  return d;
}

// MN-major (N-contiguous), 128B-swizzled B tile built from [64 k][64 n]
// TMA boxes: 64-element MN atoms 8 KiB apart (leading byte offset), 8-row K
// groups 1 KiB apart (stride byte offset) — the canonical
// ((8,n),(8,k)):((1,LBO),(8,SBO)) UMMA layout in 16-byte units.
__device__ __forceinline__ uint64_t smem_desc_mn(const void* tile) {
  const uint64_t addr = smem_addr(tile);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= uint64_t(8192 >> 4) << 16;  // LBO: next 64 columns of N
  d |= uint64_t(1024 >> 4) << 32;  // SBO: next 8 rows of K
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

template <int BN, bool kBMN, bool kAMN>
__device__ __forceinline__ constexpr uint32_t instr_desc() {
  return (1u << 4)                     // D = f32
         | (1u << 7)                   // A = bf16
         | (1u << 10)                  // B = bf16
         | (uint32_t(kAMN ? 1 : 0) << 15)  // A major: 0 = K, 1 = MN
         | (uint32_t(kBMN ? 1 : 0) << 16)  // B major: 0 = K, 1 = MN
         | (uint32_t(BN >> 3) << 17)   // N
         | (uint32_t(kBM >> 4) << 24); // M
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Whole-warp variants: every lane runs the issue loop (its state stays
// warp-uniform, so the compiler keeps descriptors in uniform registers) and
// one elected lane issues. The lane-0-only loop moved every descriptor
// through an R2UR.BROADCAST / ELECT sequence per MMA: ~25 instructions per
// MMA on one thread, which could not keep the N=128 tiles' 64-cycle MMAs
// queued (r02 SASS / ncu: tensor pipe 42% active on the pair 256x128 tile).
__device__ __forceinline__ void mma_bf16_elect(uint32_t tmem_d, uint64_t a, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// GELU with erf from Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7 on erf,
// far below bf16/fp32 output rounding): one MUFU reciprocal + one MUFU exp2
// + 8 FMAs instead of libdevice erff's ~30 instructions, so the epilogue
// keeps up with the MMAs (the GELU epilogue was the pacing stage).
__device__ __forceinline__ float gelu_erf(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = rcp_approx(1.f + 0.3275911f * z);
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  poly *= t;
  const float e = ex2_approx(-z * z * 1.4426950408889634f);
  const float erf_abs = fmaf(-poly, e, 1.f);
  const float erf_v = copysignf(erf_abs, x);
  return 0.5f * x * (1.f + erf_v);
}

// Two GELUs at once on the packed fp32x2 pipe (FFMA2 / FMUL2: one
// instruction, two lanes' worth of results), same A&S 7.1.26 erf, and with
// the reciprocal done by Newton steps on the FMA pipe instead of MUFU.RCP:
// the scalar form costs ~15 FP32 instructions + 2 MUFU per element, which
// saturates both pipes at once (0.12 clk per element per SM), so the GELU
// epilogue of a K <= 1024 GEMM ran longer than its MMAs. Here: ~10.5
// instructions + 1 MUFU (ex2) per element. GELU(x) = 0.5 (x + |x| erf(|x|/sqrt2))
// needs no copysign. The reciprocal of d = 1 + p z (d >= 1) starts from the
// exponent-reflection guess (|rel err| < 0.125) and takes three Newton steps
// (< 2.5e-7 relative, below the A&S truncation error).
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t splat2(float v) { return pk2(v, v); }

__device__ __forceinline__ void gelu_erf_x2(float& x0, float& x1) {
  const uint64_t x = pk2(x0, x1);
  const float a0 = fabsf(x0), a1 = fabsf(x1);
  const uint64_t ax = pk2(a0, a1);
  const uint64_t z = mul2(ax, splat2(0.70710678118654752f));
  const uint64_t d = fma2(z, splat2(0.3275911f), splat2(1.f));
  const uint64_t nd = fma2(z, splat2(-0.3275911f), splat2(-1.f));
  float d0, d1;
  upk2(d, d0, d1);
  uint64_t t = pk2(__int_as_float(0x7EF311C3 - __float_as_int(d0)),
                   __int_as_float(0x7EF311C3 - __float_as_int(d1)));
#pragma unroll
  for (int i = 0; i < 3; ++i) {  // t <- t (2 - d t)
    const uint64_t e = fma2(nd, t, splat2(1.f));
    t = fma2(t, e, t);
  }
  // -poly(t) (negated coefficients), so erf(|x|) = 1 + npoly * exp(-z^2)
  uint64_t q = fma2(splat2(-1.061405429f), t, splat2(1.453152027f));
  q = fma2(q, t, splat2(-1.421413741f));
  q = fma2(q, t, splat2(0.284496736f));
  q = fma2(q, t, splat2(-0.254829592f));
  q = mul2(q, t);
  const uint64_t w = mul2(mul2(z, z), splat2(-1.4426950408889634f));
  float w0, w1;
  upk2(w, w0, w1);
  const uint64_t e = pk2(ex2_approx(w0), ex2_approx(w1));
  const uint64_t ea = fma2(q, e, splat2(1.f));
  const uint64_t g = mul2(fma2(ax, ea, x), splat2(0.5f));
  upk2(g, x0, x1);
}

// Two GELU'(x) = Phi(x) + x phi(x) at once, the gelu_erf_x2 way:
// Phi(x) = 0.5 + 0.5 sign(x) erf(|x|/sqrt2), phi(x) = exp(-x^2/2)/sqrt(2 pi).
__device__ __forceinline__ uint64_t gelu_grad_x2(float x0, float x1) {
  const uint64_t x = pk2(x0, x1);
  const uint64_t z = mul2(pk2(fabsf(x0), fabsf(x1)), splat2(0.70710678118654752f));
  const uint64_t d = fma2(z, splat2(0.3275911f), splat2(1.f));
  const uint64_t nd = fma2(z, splat2(-0.3275911f), splat2(-1.f));
  float d0, d1;
  upk2(d, d0, d1);
  uint64_t t = pk2(__int_as_float(0x7EF311C3 - __float_as_int(d0)),
                   __int_as_float(0x7EF311C3 - __float_as_int(d1)));
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const uint64_t e = fma2(nd, t, splat2(1.f));
    t = fma2(t, e, t);
  }
  uint64_t q = fma2(splat2(-1.061405429f), t, splat2(1.453152027f));
  q = fma2(q, t, splat2(-1.421413741f));
  q = fma2(q, t, splat2(0.284496736f));
  q = fma2(q, t, splat2(-0.254829592f));
  q = mul2(q, t);
  const uint64_t w = mul2(mul2(z, z), splat2(-1.4426950408889634f));  // log2 exp(-x^2/2)
  float w0, w1;
  upk2(w, w0, w1);
  const uint64_t e = pk2(ex2_approx(w0), ex2_approx(w1));
  float ea0, ea1;
  upk2(fma2(q, e, splat2(1.f)), ea0, ea1);
  const uint64_t sea = pk2(copysignf(ea0, x0), copysignf(ea1, x1));
  const uint64_t phi_half = fma2(sea, splat2(0.5f), splat2(0.5f));
  return fma2(mul2(x, splat2(0.3989422804014327f)), e, phi_half);
}

// d/dx GELU(x) = Phi(x) + x phi(x), with the same A&S erf as gelu_erf.
__device__ __forceinline__ float gelu_grad(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float t = rcp_approx(1.f + 0.3275911f * z);
  float poly = fmaf(1.061405429f, t, -1.453152027f);
  poly = fmaf(poly, t, 1.421413741f);
  poly = fmaf(poly, t, -0.284496736f);
  poly = fmaf(poly, t, 0.254829592f);
  poly *= t;
  const float e = ex2_approx(-z * z * 1.4426950408889634f);  // exp(-x^2 / 2)
  const float erf_v = copysignf(fmaf(-poly, e, 1.f), x);
  return 0.5f * (1.f + erf_v) + x * e * 0.3989422804014327f;
}

// Epilogues: 0 = none, 1 = GELU, 2 = GELU backward (C = acc * GELU'(aux),
// aux bf16 [M, N] with leading dimension ldaux: the saved pre-activation).
constexpr int kEpiNone = 0, kEpiGelu = 1, kEpiDGelu = 2;

constexpr int kEpiGeluSave = 3;  // GELU, and the pre-activation stored to aux (training)

// 32 accumulator columns of one row: epilogue computed once, then stored to
// each of `fan` outputs (the fused all-reduce writes every group member).
// Vector path when the 32 columns are in bounds and 16-byte aligned.
// The epilogue's arithmetic on 32 accumulator columns of one row, in place:
// GELU backward against aux, the pre-activation saved to aux, GELU.
template <int kEpi>
__device__ __forceinline__ void epi_values32(float (&v)[32], int row, int col, int M, int N,
                                             const void* aux, int ldaux) {
  if (row >= M || col >= N) return;
  const bool full = col + 32 <= N;
  if constexpr (kEpi == kEpiDGelu) {
    const __nv_bfloat16* a =
        static_cast<const __nv_bfloat16*>(aux) + static_cast<size_t>(row) * ldaux + col;
    if (full && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = reinterpret_cast<const uint4*>(a)[q];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(h[i]);
          float g0, g1;
          upk2(mul2(pk2(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]), gelu_grad_x2(f.x, f.y)), g0, g1);
          v[8 * q + 2 * i] = g0;
          v[8 * q + 2 * i + 1] = g1;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col + i < N) v[i] *= gelu_grad(__bfloat162float(a[i]));
    }
  }
  if constexpr (kEpi == kEpiGeluSave) {  // pre-activation out (bf16), before GELU
    __nv_bfloat16* a = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(aux)) +
                       static_cast<size_t>(row) * ldaux + col;
    if (full && (reinterpret_cast<uintptr_t>(a) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t p[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]);
          std::memcpy(&p[i], &h, 4);
        }
        reinterpret_cast<uint4*>(a)[q] = make_uint4(p[0], p[1], p[2], p[3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col + i < N) a[i] = __float2bfloat16_rn(v[i]);
    }
  }
  if constexpr (kEpi == kEpiGelu || kEpi == kEpiGeluSave) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) gelu_erf_x2(v[i], v[i + 1]);
  }
}

template <int kEpi, bool kOutF32>
__device__ __forceinline__ void epi_store32(void* const* outs, int fan, int ldc, int M, int N,
                                            int row, int col, const uint32_t (&r)[32],
                                            const void* aux, int ldaux) {
  if (row >= M || col >= N) return;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  epi_values32<kEpi>(v, row, col, M, N, aux, ldaux);
  const bool full = col + 32 <= N;
  if constexpr (kOutF32) {
    for (int j = 0; j < fan; ++j) {
      float* dst = static_cast<float*>(outs[j]) + static_cast<size_t>(row) * ldc + col;
      if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      } else {
        for (int i = 0; i < 32; ++i)
          if (col + i < N) dst[i] = v[i];
      }
    }
  } else {
    uint32_t p[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      std::memcpy(&p[i], &h, 4);
    }
    for (int j = 0; j < fan; ++j) {
      __nv_bfloat16* dst =
          static_cast<__nv_bfloat16*>(outs[j]) + static_cast<size_t>(row) * ldc + col;
      if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          reinterpret_cast<uint4*>(dst)[q] = make_uint4(p[4 * q], p[4 * q + 1], p[4 * q + 2],
                                                        p[4 * q + 3]);
      } else {
        for (int i = 0; i < 32; ++i)
          if (col + i < N) dst[i] = __float2bfloat16_rn(v[i]);
      }
    }
  }
}

// ---- TMA-store epilogue ---------------------------------------------------
// Each epilogue warp stages 32 rows x 128 bytes of output (64 bf16 / 32 fp32
// columns) in its own 4 KiB of shared memory, 128B-swizzled (16-byte vector
// q of row r at q ^ (r % 8): the warp's row-per-lane stores are bank-conflict
// free), and one lane writes the box to every fan-out output with
// cp.async.bulk.tensor stores (out-of-bounds rows / columns clipped by TMA).
// The per-lane st.global epilogue scattered 32 rows per instruction, which
// paced the small-K GEMMs (r02 ncu: the MMA pipe idled behind it).
constexpr int kStageOut = 4096;                  // per epilogue warp
constexpr int kStagingBytes = kEpiWarps * kStageOut;

template <bool kOutF32>
__device__ __forceinline__ void epi_stage32(uint8_t* stage, int lane, int piece,
                                            const float (&v)[32]) {
  uint8_t* row = stage + lane * 128;
  if constexpr (kOutF32) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<float4*>(row + ((q ^ (lane & 7)) << 4)) =
          make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t p[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]);
        std::memcpy(&p[i], &h, 4);
      }
      *reinterpret_cast<uint4*>(row + (((4 * piece + q) ^ (lane & 7)) << 4)) =
          make_uint4(p[0], p[1], p[2], p[3]);
    }
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x,
                                             int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_addr(src)), "r"(x), "r"(y)
      : "memory");
}

// ---- stream-K / split-K fixup through TMA -------------------------------------
// The fp32 partial tiles live in sk_ws, viewed by args.skmap as
// [CTAs x 128 rows][BN cols] (32 x 32 fp32 boxes, 128B swizzle). A partial
// CTA's warp stages its 32 rows x 32 columns and bulk-stores them; the head
// TMA-loads each later CTA's box into the same staging and adds it from
// shared memory. The per-lane float4 form scattered 32 rows per instruction
// (~8k L2 requests per CTA each way) and made every split slower than whole
// tiles (profiles/r02_gemm_sweep_split.jsonl).
__device__ __forceinline__ void sk_store_chunk(const CUtensorMap* map, uint8_t* stage, int lane,
                                               const uint32_t (&r)[32], int col, int row) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  epi_stage32<true>(stage, lane, 0, v);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(map, stage, col, row);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}
// every partial box written and visible (generic and async proxies) before
// the CTA's flag is released
__device__ __forceinline__ void sk_store_done(int lane) {
  if (lane == 0)
    asm volatile("cp.async.bulk.wait_group 0;\n\tfence.proxy.async.global;" ::: "memory");
  __syncwarp();
}
// head: r += the 32 x 32 fp32 box of a partial tile at (col, row); the
// staging must be free (no bulk store still reading it)
__device__ __forceinline__ void sk_add_chunk(const CUtensorMap* map, uint8_t* stage,
                                             uint64_t* bar, uint32_t& phase, int lane,
                                             uint32_t (&r)[32], int col, int row) {
  if (lane == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(bar, 32 * 128);
    tma_load_2d(stage, map, bar, col, row);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
  const uint8_t* rowp = stage + lane * 128;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 p = *reinterpret_cast<const float4*>(rowp + ((q ^ (lane & 7)) << 4));
    r[4 * q] = __float_as_uint(__uint_as_float(r[4 * q]) + p.x);
    r[4 * q + 1] = __float_as_uint(__uint_as_float(r[4 * q + 1]) + p.y);
    r[4 * q + 2] = __float_as_uint(__uint_as_float(r[4 * q + 2]) + p.z);
    r[4 * q + 3] = __float_as_uint(__uint_as_float(r[4 * q + 3]) + p.w);
  }
  __syncwarp();  // every lane read the box before the next load overwrites it
}

// Programmatic dependent launch: everything above this point (barrier init,
// TMEM allocation, tensor-map prefetch) overlaps the previous kernel's tail;
// no global memory is touched before the wait, which returns once the
// prerequisite grid has completed and its writes are visible. The dependents
// are released at once: the grid is persistent, so every CTA is resident by
// the time all have executed this. Both are no-ops without the launch
// attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int BN>
struct Smem {
  static constexpr int kStageA = kBM * kBK * 2;
  static constexpr int kStageB = BN * kBK * 2;
  static constexpr int kStages = (BN >= 256) ? 4 : 6;
  static constexpr int kData = kStages * (kStageA + kStageB);
  // [stage ring][output staging, 1024-aligned][barriers]
  static constexpr int kBytes = kData + kStagingBytes + 1024 /*align slack*/ + 256 /*barriers*/;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Persistent: CTA b handles tiles b, b + grid, ... (n fastest). The MMA of
// tile i+1 overlaps the epilogue of tile i through two TMEM accumulators.
// kBMN: B is the logical row-major [K, N] (N contiguous, MN-major operand)
// instead of Bt [N, K].
// A batch of equally shaped problems (one per simulated device of a mesh)
// shares one persistent launch: tiles of all problems form one work list,
// so small per-device GEMMs do not each pay a partial last wave.
constexpr int kMaxBatch = 8;
//
// Fused reduction (simulated-mesh partial sums): output problem g sums
// `reduce` inputs (maps a/b[g*reduce + r]) into one TMEM accumulator — the
// k-loop simply runs over every input's K blocks — and the epilogue writes
// the finished tile to `fan` outputs (c[g*fan + j]). With reduce = fan =
// group size this is the split-k GEMM and its all-reduce in one kernel:
// no partial buffers, no reduction pass, every replica bit-identical.
//
// kAMN: A is given transposed, as the row-major [K, M] (M contiguous, an
// MN-major UMMA operand) -- the weight-gradient GEMM dW = X^T . dY reads the
// saved activation X [tokens, features] as is, with no transpose pass.
struct GemmArgs {
  CUtensorMap a[kMaxBatch];
  CUtensorMap b[kMaxBatch];
  void* c[kMaxBatch];
  const void* aux[kMaxBatch];  // kEpiDGelu: pre-activation per output problem
  int count, M, N, K, ldc, ldaux;
  int reduce, fan;
  // > 0: fused reduce-scatter epilogue (single problem). Rows are owned in
  // blocks of scatter_rows; a tile's rows go to c[owner] (the owner's
  // staging slab for this rank, typically a peer-mapped pointer), so the
  // partial tile crosses NVLink while the next tile's MMAs run.
  int scatter_rows;
  // Stream-K (single-CTA kernel, reduce == fan == 1): CTA b owns the
  // k-iterations [b*T/G, (b+1)*T/G) of the tile-major iteration space, so an
  // under-filled problem keeps every SM busy. A tile split across CTAs is
  // finished by the CTA holding its first k-block (the "head", at the end of
  // its range); the others (at the start of theirs) write fp32 partial tiles
  // to sk_ws[cta] and raise sk_flags[cta]; the head adds them in CTA order
  // (deterministic) and clears the flags.
  int streamk;
  float* sk_ws;
  int* sk_flags;
  // TMA-store epilogue: cmap[g * fan + j] maps output c[g * fan + j]
  // (box 32 rows x 128 bytes, 128B swizzle); 0 = per-lane st.global stores
  // (scatter_rows, unaligned outputs).
  int tma_out;
  int sk_tma;             // stream-K fixup through args.skmap (TMA) instead of per-lane
  CUtensorMap skmap;      // fp32 view of sk_ws: [CTAs x 128][BN]
  int sk_units;  // > 0: stream-K grid of exactly this many CTAs / clusters (aligned split-K)
  // pair kernel: 4-CTA clusters multicasting A across two pairs (A maps with
  // 64-row boxes)
  int a_mc;
  // diagnostics (apl_gemm_trace): per-CTA timestamps of the kernel's phases,
  // kTraceSlots per CTA; nullptr in normal runs
  unsigned long long* trace;
  int trace_ctas;  // CTAs the trace buffer holds (kTraceSlots u64 each)
  CUtensorMap cmap[kMaxBatch];
};

constexpr int kTraceSlots = 16;
// slot 0: %globaltimer at entry; 1..: clock64 at entry, after the prologue,
// after griddepcontrol.wait, first TMA issued, first stage landed (MMA
// issuer), last accumulator committed, last accumulator drained by epilogue
// warp 0, its last store issued, its bulk stores done, teardown start, exit
__device__ __forceinline__ void trace_mark(unsigned long long* trace, int slot) {
  if (trace != nullptr) {  // launches only trace when the buffer covers the grid
    long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    trace[blockIdx.x * kTraceSlots + slot] = static_cast<unsigned long long>(c);
  }
}

// Segments of the (tile, k-block) iteration space a CTA processes, in order.
struct SegIter {
  int64_t pos, end, total;
  int t, tiles, grid, KT;
  bool sk;
  __device__ SegIter(bool streamk, int b, int G, int tiles_, int KT_)
      : tiles(tiles_), grid(G), KT(KT_), sk(streamk) {
    total = static_cast<int64_t>(tiles_) * KT_;
    pos = sk ? total * b / G : 0;
    end = sk ? total * (b + 1) / G : 0;
    t = b;
  }
  __device__ bool next(int& tile, int& k0, int& k1) {
    if (sk) {
      if (pos >= end) return false;
      tile = static_cast<int>(pos / KT);
      k0 = static_cast<int>(pos - static_cast<int64_t>(tile) * KT);
      const int64_t left = end - pos;
      k1 = left < KT - k0 ? k0 + static_cast<int>(left) : KT;
      pos += k1 - k0;
      return true;
    }
    if (t >= tiles) return false;
    tile = t;
    k0 = 0;
    k1 = KT;
    t += grid;
    return true;
  }
};

template <int BN, int kEpi, bool kOutF32, bool kBMN, bool kAMN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05(const __grid_constant__ GemmArgs args) {
  const int M = args.M, N = args.N, K = args.K, ldc = args.ldc;
  using S = Smem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* tiles_a = base;
  uint8_t* tiles_b = base + S::kStages * S::kStageA;
  uint8_t* staging = base + S::kData;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S::kData + kStagingBytes);
  uint64_t* empty = full + S::kStages;
  uint64_t* acc_full = empty + S::kStages;  // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2;       // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint64_t* pbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [kEpiWarps] stream-K loads

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int kblocks = (K + kBK - 1) / kBK;
  const int n_tiles = (N + BN - 1) / BN;
  const int per_problem = ((M + kBM - 1) / kBM) * n_tiles;
  const int tiles = per_problem * args.count;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kEpiWarps);  // one arrive per epilogue warp
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&pbar[w], 1);  // stream-K box loads
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int g = 0; g < args.count * args.reduce; ++g) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&args.a[g])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&args.b[g])) : "memory");
    }
  }
  if (warp == 1) {  // whole warp allocates 2 x BN fp32 columns of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(S::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_enter();

  const int KT = kblocks * args.reduce;
  if (warp == 0) {
    // TMA producer: the whole warp walks the schedule (warp-uniform state,
    // no per-K-block division: the input slice r and its block kb advance
    // incrementally), one elected lane issues
    {
      int it = 0;  // ring position across tiles
      SegIter seg(args.streamk != 0, blockIdx.x, gridDim.x, tiles, KT);
      int t, k0, k1;
      while (seg.next(t, k0, k1)) {
        const int g = t / per_problem, lt = t % per_problem;
        const int m0 = (lt / n_tiles) * kBM, n0 = (lt % n_tiles) * BN;
        int r = k0 / kblocks, kb = k0 - r * kblocks;
        for (int kk = k0; kk < k1; ++kk, ++it) {
          const CUtensorMap* map_a = &args.a[g * args.reduce + r];
          const CUtensorMap* map_b = &args.b[g * args.reduce + r];
          const int s = it % S::kStages;
          const uint32_t phase = (it / S::kStages) & 1;
          mbar_wait(&empty[s], phase ^ 1);
          mbar_expect_tx_e(&full[s], S::kStageA + S::kStageB);
          if constexpr (kAMN) {
            // two boxes of [64 k][64 m], one MN swizzle atom column each
            tma_load_2d_e(tiles_a + s * S::kStageA, map_a, &full[s], m0, kb * kBK);
            tma_load_2d_e(tiles_a + s * S::kStageA + 8192, map_a, &full[s], m0 + 64, kb * kBK);
          } else {
            tma_load_2d_e(tiles_a + s * S::kStageA, map_a, &full[s], kb * kBK, m0);
          }
          if constexpr (kBMN) {
            // BN/64 boxes of [64 k][64 n], one MN swizzle atom column each
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d_e(tiles_b + s * S::kStageB + j * 8192, map_b, &full[s], n0 + j * 64,
                            kb * kBK);
          } else {
            tma_load_2d_e(tiles_b + s * S::kStageB, map_b, &full[s], kb * kBK, n0);
          }
          if (++kb == kblocks) {
            kb = 0;
            ++r;
          }
        }
      }
    }
  } else if (warp == 1) {
    // MMA issuer: the whole warp walks the schedule, one elected lane issues
    {
      constexpr uint32_t idesc = instr_desc<BN, kBMN, kAMN>();
      const uint64_t da0 = kAMN ? smem_desc_mn(tiles_a) : smem_desc(tiles_a);
      const uint64_t db0 = kBMN ? smem_desc_mn(tiles_b) : smem_desc(tiles_b);
      int it = 0, local = 0;
      SegIter seg(args.streamk != 0, blockIdx.x, gridDim.x, tiles, KT);
      int t, k0, k1;
      for (; seg.next(t, k0, k1); ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);  // epilogue drained this buffer
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kk = k0; kk < k1; ++kk, ++it) {
          const int s = it % S::kStages;
          const uint32_t phase = (it / S::kStages) & 1;
          mbar_wait(&full[s], phase);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          // stage s's descriptors: base + s stages (address field in 16 B units)
          const uint64_t da = da0 + uint64_t(s) * (S::kStageA >> 4);
          const uint64_t db = db0 + uint64_t(s) * (S::kStageB >> 4);
          // K advance per instruction: K-major = 32 B inside the swizzle row;
          // MN-major = 16 rows of 128 B.
          constexpr uint64_t kAdvA = kAMN ? (16 * 128) >> 4 : 2;
          constexpr uint64_t kAdvB = kBMN ? (16 * 128) >> 4 : 2;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            mma_bf16_elect(d, da + kAdvA * k, db + kAdvB * k, idesc,
                           (kk > k0 || k > 0) ? 1u : 0u);
          }
          mma_commit_elect(&empty[s]);  // frees the slot once these MMAs have read it
        }
        mma_commit_elect(&acc_full[acc]);  // accumulator complete
      }
    }
  } else {
    // Epilogue warps 2..9 -> TMEM lane quarter (warp % 4), half the columns each.
    const int quarter = warp % 4;          // TMEM lanes this warp may access
    const int half = (warp - 2) / 4;       // which half of the tile's columns
    int local = 0;
    uint32_t pphase = 0;  // this warp's stream-K box-load barrier phase
    SegIter seg(args.streamk != 0, blockIdx.x, gridDim.x, tiles, KT);
    int t, k0, k1;
    for (; seg.next(t, k0, k1); ++local) {
      const int acc = local & 1;
      const int g = t / per_problem, lt = t % per_problem;
      const int m0 = (lt / n_tiles) * kBM, n0 = (lt % n_tiles) * BN;
      void* const* outs = args.c + g * args.fan;
      const int trow = quarter * 32 + lane;  // row within the tile
      int row = m0 + trow;
      int rows = M, fan = args.fan;
      if (args.scatter_rows > 0) {
        const int owner = m0 / args.scatter_rows;
        outs = args.c + owner;
        row -= owner * args.scatter_rows;
        rows = args.scatter_rows;
        fan = 1;
      }
      // stream-K roles: partial (k0 > 0: write fp32 tile for the head) or
      // head of a split tile (k0 == 0, k1 < KT: add the later CTAs' partials)
      const bool partial = k0 > 0;
      const bool head = !partial && k1 < KT;
      int c_first = 0, c_last = -1;
      if (head) {
        // CTAs after this one whose ranges start inside this tile
        // (CTAs with empty ranges contribute nothing and raise no flag)
        const int64_t tile_end = static_cast<int64_t>(t + 1) * KT;
        const int G = gridDim.x;
        c_first = blockIdx.x + 1;
        c_last = blockIdx.x;
        while (c_last + 1 < G && seg.total * (c_last + 1) / G < tile_end) ++c_last;
        for (int c = c_first; c <= c_last; ++c) {
          if (seg.total * c / G == seg.total * (c + 1) / G) continue;  // empty range
          volatile int* f = args.sk_flags + c;
          while (true) {
            int v;
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if (v != 0) break;
            __nanosleep(64);
          }
        }
      }
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      // head of a split tile, per-lane form: partial of CTA cc, columns [c, c+32)
      auto add_one = [&](uint32_t (&r)[32], int c, int cc) {
        const float4* w = reinterpret_cast<const float4*>(
            args.sk_ws + (static_cast<size_t>(cc) * kBM + trow) * BN + c);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 p = w[i];
          r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + p.x);
          r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + p.y);
          r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + p.z);
          r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + p.w);
        }
      };
      // head of a split tile: add the later CTAs' fp32 partials of columns [c, c+32)
      auto add_parts = [&](uint32_t (&r)[32], int c) {
        for (int cc = c_first; cc <= c_last; ++cc) {
          if (seg.total * cc / gridDim.x == seg.total * (cc + 1) / gridDim.x) continue;
          const float4* w = reinterpret_cast<const float4*>(
              args.sk_ws + (static_cast<size_t>(cc) * kBM + trow) * BN + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 p = w[i];
            r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + p.x);
            r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + p.y);
            r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + p.z);
            r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + p.w);
          }
        }
      };
      uint8_t* stage = staging + (warp - 2) * kStageOut;
      if (partial && args.sk_tma) {  // raw accumulator to this CTA's partial tile
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
          uint32_t r[32];
          tmem_ld32(lane_addr + uint32_t(c), r);
          sk_store_chunk(&args.skmap, stage, lane, r, c, static_cast<int>(blockIdx.x) * kBM + quarter * 32);
        }
        sk_store_done(lane);
      } else if (args.tma_out && !partial) {
        constexpr int kCW = kOutF32 ? 32 : 64;  // columns per 128-byte staged row
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += kCW) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();  // the previous box's store has read the staging
          uint32_t r[kCW / 32][32];
#pragma unroll
          for (int p = 0; p < kCW / 32; ++p) tmem_ld32(lane_addr + uint32_t(c + 32 * p), r[p]);
          if (head) {  // add the later CTAs' partials, in CTA order (deterministic)
            for (int cc = c_first; cc <= c_last; ++cc) {
              if (seg.total * cc / gridDim.x == seg.total * (cc + 1) / gridDim.x) continue;
#pragma unroll
              for (int p = 0; p < kCW / 32; ++p) {
                if (args.sk_tma)
                  sk_add_chunk(&args.skmap, stage, &pbar[warp - 2], pphase, lane, r[p],
                               c + 32 * p, cc * kBM + quarter * 32);
                else
                  add_one(r[p], c + 32 * p, cc);
              }
            }
          }
#pragma unroll
          for (int p = 0; p < kCW / 32; ++p) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[p][i]);
            epi_values32<kEpi>(v, row, n0 + c + 32 * p, rows, N, args.aux[g], args.ldaux);
            epi_stage32<kOutF32>(stage, lane, p, v);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            for (int j = 0; j < fan; ++j)
              tma_store_2d(&args.cmap[g * args.fan + j], stage, n0 + c, m0 + quarter * 32);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      } else {
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
        uint32_t r[32];
        tmem_ld32(lane_addr + uint32_t(c), r);
        if (partial) {
          float4* w = reinterpret_cast<float4*>(args.sk_ws +
                                                (static_cast<size_t>(blockIdx.x) * kBM + trow) * BN + c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                               __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          continue;
        }
        add_parts(r, c);
        epi_store32<kEpi, kOutF32>(outs, fan, ldc, rows, N, row, n0 + c, r, args.aux[g],
                                   args.ldaux);
      }
      }
      // All TMEM reads of this buffer are done: hand it back to the MMA warp.
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (partial || head) {
        // all 8 epilogue warps finished writing (partial) / reading (head)
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (warp == 2 && lane == 0) {
          if (partial) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(args.sk_flags + blockIdx.x),
                         "r"(1)
                         : "memory");
          } else {
            for (int cc = c_first; cc <= c_last; ++cc) args.sk_flags[cc] = 0;
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(S::kTmemCols));
  }
}

// ---- 2-CTA (CTA pair) variant: tcgen05.mma.cta_group::2, M = 256 ----------
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile: CTA r loads
// rows [r*128, r*128+128) of A and rows/columns [r*128, r*128+128) of B
// into the same shared-memory offsets, the leader (rank 0) issues
// M=256,N=256 MMAs that read both CTAs' operand halves, and each CTA's
// TMEM receives its own 128 accumulator rows. Per SM this halves the B
// operand traffic of the 1-CTA 128 x 256 tile (32 KiB instead of 48 KiB of
// shared-memory fill per 64-deep K block), which is what limits it.
//
// Barrier protocol (same shared-memory offsets in both CTAs):
//   full[s]      leader only, count 2: leader arrive.expect_tx(both CTAs'
//                bytes) + peer's remote arrive; both CTAs' TMA loads
//                complete_tx on the leader's barrier (peer bit cleared).
//   empty[s]     per CTA, count 1: leader's tcgen05.commit multicast (0b11).
//   acc_full[a]  per CTA, count 1: leader's commit multicast after the tile.
//   acc_empty[a] leader only, count 8: 4 epilogue warps x 2 CTAs arrive
//                (peer through mapa) once their TMEM rows are read.
namespace pair {

constexpr int kBM = 128;  // rows per CTA (M = 256 per pair)

// Pair tile 256 x BN: each CTA stages its 128 rows of A and BN/2 rows (or
// columns) of B per 64-deep K block; the MMA reads both CTAs' B halves.
template <int BN>
struct Cfg {
  static constexpr int kStageA = kBM * kBK * 2;         // 16 KiB
  static constexpr int kStageB = (BN / 2) * kBK * 2;    // 8 / 16 KiB
  static constexpr int kStages = BN >= 256 ? 6 : 8;
  static constexpr int kData = kStages * (kStageA + kStageB);
  static constexpr int kBytes = kData + kStagingBytes + 1024 + 256;
  static constexpr int kTmemCols = 2 * BN;  // double-buffered fp32 accumulator
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr_local, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(saddr_local), "r"(rank));
  return out;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void remote_arrive(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// TMA load whose completion is counted on the leader CTA's barrier.
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map,
                                                 uint64_t* bar_local, int x, int y) {
  const uint32_t bar = smem_addr(bar_local) & 0xFEFFFFFFu;  // peer bit -> rank 0
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

// Elected-lane forms for the whole-warp pair producer.
__device__ __forceinline__ void tma_load_2d_pair_e(void* dst, const CUtensorMap* map,
                                                   uint64_t* bar_local, int x, int y) {
  const uint32_t bar = smem_addr(bar_local) & 0xFEFFFFFFu;  // peer bit -> rank 0
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n}\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_mc_e(void* dst, const CUtensorMap* map,
                                                      uint64_t* bar_local, int x, int y,
                                                      uint16_t mask) {
  const uint32_t bar = smem_addr(bar_local) & 0xFEFFFFFFu;
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;\n}\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void remote_arrive_e(uint32_t cluster_addr) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.shared::cluster.b64 _, [%0];\n}\n" ::"r"(cluster_addr)
      : "memory");
}

// Multicast variant: the box lands at the same offset in every CTA of `mask`,
// each destination's completion counted on its pair leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const CUtensorMap* map,
                                                    uint64_t* bar_local, int x, int y,
                                                    uint16_t mask) {
  const uint32_t bar = smem_addr(bar_local) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_pair_elect(uint32_t tmem_d, uint64_t a, uint64_t b,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit_pair_elect(uint64_t* bar_local, uint16_t mask) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n"
      "}\n" ::"r"(smem_addr(bar_local)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void commit_pair(uint64_t* bar_local, uint16_t mask = 0b11) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_addr(bar_local)),
      "h"(mask)
      : "memory");
}

template <int BN, bool kBMN, bool kAMN>
__device__ __forceinline__ constexpr uint32_t instr_desc_pair() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kAMN ? 1 : 0) << 15) |
         (uint32_t(kBMN ? 1 : 0) << 16) |
         (uint32_t(BN >> 3) << 17) | (uint32_t((2 * kBM) >> 4) << 24);
}

// Spin on a stream-K partial flag (acquire), trapping after ~4 s instead of
// hanging the GPU if the writer can never run.
__device__ __forceinline__ void wait_flag(const int* f) {
  const long long t0 = clock64();
  while (true) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v != 0) return;
    __nanosleep(64);
    if (clock64() - t0 > (1ll << 33)) __trap();
  }
}

// Persistent over pair tiles (cluster c takes tiles c, c + clusters, ...),
// or -- args.streamk -- over a contiguous range of the (tile, k-block)
// iteration space: cluster c owns [c*T/G, (c+1)*T/G). A tile split across
// clusters is finished by the cluster holding its first k-block (its range
// ENDS inside the tile: the "head"); each later cluster (its range STARTS
// inside the tile) writes its fp32 partial -- each CTA its own 128 rows --
// to sk_ws[its CTA] and raises sk_flags[its CTA]; the head CTA of the same
// cluster rank adds them in cluster order (deterministic) and clears them.
//
// kMC: a cluster of 4 = two CTA pairs on adjacent N tiles of the same 256
// rows. Both pairs need the same A rows, so each CTA loads half of its 128
// A rows and multicasts them to its counterpart in the other pair: L2 reads
// per SM drop from (A 16 + B 8|16) to (A 8 + B 8|16) KiB per 64-deep K
// block, the operand fill that paced the pair kernel. A stage is refilled
// only when both pairs' MMAs have freed it (empty[] counts both leaders'
// commits). Whole N-tile pairs only (host: even tile count, no stream-K).
template <int BN, int kEpi, bool kOutF32, bool kBMN, bool kAMN, bool kMC>
__global__ void __cluster_dims__(kMC ? 4 : 2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_bf16_tcgen05_pair(const __grid_constant__ GemmArgs args) {
  using S = Cfg<BN>;
  if (args.trace != nullptr && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    args.trace[blockIdx.x * kTraceSlots] = g;
    trace_mark(args.trace, 1);
  }
  const int M = args.M, N = args.N, K = args.K, ldc = args.ldc;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* tiles_a = base;
  uint8_t* tiles_b = base + S::kStages * S::kStageA;
  uint8_t* staging = base + S::kData;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S::kData + kStagingBytes);
  uint64_t* empty = full + S::kStages;
  uint64_t* acc_full = empty + S::kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint64_t* pbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // [kEpiWarps] stream-K loads

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int kCS = kMC ? 4 : 2;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1u;  // position in the CTA pair (0: MMA leader)
  const int pid = static_cast<int>(crank >> 1);  // pair within a kMC cluster
  const uint32_t pair_leader = crank & ~1u;
  const bool leader = rank == 0;
  const int kblocks = (K + kBK - 1) / kBK;
  const int n_tiles = (N + BN - 1) / BN;
  const int n_units = kMC ? n_tiles / 2 : n_tiles;  // N tiles (pairs of them) per cluster tile
  const int per_problem = ((M + 2 * kBM - 1) / (2 * kBM)) * n_units;
  const int tiles = per_problem * args.count;
  const int cluster = blockIdx.x / kCS, clusters = gridDim.x / kCS;
  auto ntile_of = [&](int lt) { return kMC ? (lt % n_units) * 2 + pid : lt % n_units; };
  const int KT = kblocks * args.reduce;
  const bool sk = args.streamk != 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S::kStages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], kMC ? 2 : 1);  // kMC: both pair leaders' commits
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * kEpiWarps);  // epilogue warps of both CTAs
    }
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&pbar[w], 1);  // stream-K box loads
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int g = 0; g < args.count * args.reduce; ++g) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&args.a[g])) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&args.b[g])) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(S::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // barriers initialised in both CTAs before any remote use: the
  // fence.mbarrier_init.release.cluster above already publishes them, so the
  // arrive is relaxed (no MEMBAR.GPU / ERRBAR drain in the prologue)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) trace_mark(args.trace, 2);
  pdl_enter();
  if (threadIdx.x == 0) trace_mark(args.trace, 3);

  if (warp == 0) {
    // TMA producer: whole warp, incremental K position, one elected lane issues
    {
      const uint32_t full_leader0 = map_to_rank(smem_addr(&full[0]), pair_leader);
      const uint16_t a_mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
      int it = 0;
      SegIter seg(sk, cluster, clusters, tiles, KT);
      int t, k0, k1;
      if (lane == 0) trace_mark(args.trace, 4);  // producer about to enter its loop
      while (seg.next(t, k0, k1)) {
        const int g = t / per_problem, lt = t % per_problem;
        const int m0 = (lt / n_units) * 2 * kBM + static_cast<int>(rank) * kBM;
        const int n0 = ntile_of(lt) * BN + static_cast<int>(rank) * (BN / 2);
        int r = k0 / kblocks, kb = k0 - r * kblocks;
        for (int kk = k0; kk < k1; ++kk, ++it) {
          const CUtensorMap* map_a = &args.a[g * args.reduce + r];
          const CUtensorMap* map_b = &args.b[g * args.reduce + r];
          const int s = it % S::kStages;
          const uint32_t phase = (it / S::kStages) & 1;
          mbar_wait(&empty[s], phase ^ 1);
          if (leader) mbar_expect_tx_e(&full[s], 2 * (S::kStageA + S::kStageB));
          if constexpr (kMC) {  // this CTA's 64-row half of the A rows, to both pairs
            if constexpr (kAMN)
              tma_load_2d_pair_mc_e(tiles_a + s * S::kStageA + pid * 8192, map_a, &full[s],
                                    m0 + pid * 64, kb * kBK, a_mask);
            else
              tma_load_2d_pair_mc_e(tiles_a + s * S::kStageA + pid * 8192, map_a, &full[s],
                                    kb * kBK, m0 + pid * 64, a_mask);
          } else if constexpr (kAMN) {  // A^T stored [K, M]: two [64 k][64 m] MN atoms
            tma_load_2d_pair_e(tiles_a + s * S::kStageA, map_a, &full[s], m0, kb * kBK);
            tma_load_2d_pair_e(tiles_a + s * S::kStageA + 8192, map_a, &full[s], m0 + 64,
                               kb * kBK);
          } else {
            tma_load_2d_pair_e(tiles_a + s * S::kStageA, map_a, &full[s], kb * kBK, m0);
          }
          if constexpr (kBMN) {
#pragma unroll
            for (int j = 0; j < (BN / 2) / 64; ++j)
              tma_load_2d_pair_e(tiles_b + s * S::kStageB + j * 8192, map_b, &full[s],
                                 n0 + j * 64, kb * kBK);
          } else {
            tma_load_2d_pair_e(tiles_b + s * S::kStageB, map_b, &full[s], kb * kBK, n0);
          }
          if (!leader) remote_arrive_e(full_leader0 + s * 8);
          if (++kb == kblocks) {
            kb = 0;
            ++r;
          }
        }
      }
      // drain: the issuer's stage-release commits land in this CTA's empty
      // barriers (both CTAs of the pair, and the other pair's with kMC); wait
      // for the last ones so none is in flight at teardown
      for (int j = 0; j < S::kStages && j < it; ++j) {
        const int i2 = it - 1 - j;
        mbar_wait(&empty[i2 % S::kStages], (i2 / S::kStages) & 1);
      }
    }
  } else if (warp == 1) {
    if (leader) {  // whole warp walks the schedule, one elected lane issues
      constexpr uint32_t idesc = instr_desc_pair<BN, kBMN, kAMN>();
      const uint64_t da0 = kAMN ? smem_desc_mn(tiles_a) : smem_desc(tiles_a);
      const uint64_t db0 = kBMN ? smem_desc_mn(tiles_b) : smem_desc(tiles_b);
      int it = 0, local = 0;
      SegIter seg(sk, cluster, clusters, tiles, KT);
      int t, k0, k1;
      if (lane == 0) trace_mark(args.trace, 5);  // issuer about to enter its loop
      for (; seg.next(t, k0, k1); ++local) {
        const int acc = local & 1;
        mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + uint32_t(acc * BN);
        for (int kk = k0; kk < k1; ++kk, ++it) {
          const int s = it % S::kStages;
          mbar_wait(&full[s], (it / S::kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t da = da0 + uint64_t(s) * (S::kStageA >> 4);
          const uint64_t db = db0 + uint64_t(s) * (S::kStageB >> 4);
          constexpr uint64_t kAdvA = kAMN ? (16 * 128) >> 4 : 2;
          constexpr uint64_t kAdvB = kBMN ? (16 * 128) >> 4 : 2;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_pair_elect(d, da + kAdvA * k, db + kAdvB * k, idesc,
                           (kk > k0 || k > 0) ? 1u : 0u);
          commit_pair_elect(&empty[s], kMC ? 0b1111 : 0b11);  // kMC: the other pair's stage too
        }
        commit_pair_elect(&acc_full[acc], static_cast<uint16_t>(0b11u << (2 * pid)));
        if (lane == 0) trace_mark(args.trace, 6);
      }
    }
  } else {
    const int quarter = warp % 4;
    const int half = (warp - 2) / 4;
    const uint32_t acc_empty_leader = map_to_rank(smem_addr(&acc_empty[0]), pair_leader);
    // accumulator-release arrivals for this cluster's last two tiles are never
    // waited on (the MMA issuer waits on tile l-2's before tile l); skipping
    // them leaves no remote arrive in flight at teardown
    int ntiles = 0;
    {
      SegIter cnt(sk, cluster, clusters, tiles, KT);
      int a0, a1, a2;
      while (cnt.next(a0, a1, a2)) ++ntiles;
    }
    int local = 0;
    uint32_t pphase = 0;  // this warp's stream-K box-load barrier phase
    SegIter seg(sk, cluster, clusters, tiles, KT);
    int t, k0, k1;
    for (; seg.next(t, k0, k1); ++local) {
      const int acc = local & 1;
      const int g = t / per_problem, lt = t % per_problem;
      const int m0 = (lt / n_units) * 2 * kBM + static_cast<int>(rank) * kBM;
      const int n0 = ntile_of(lt) * BN;
      void* const* const outs = args.c + g * args.fan;
      const int trow = quarter * 32 + lane;
      const int row = m0 + trow;
      const bool partial = k0 > 0;
      const bool head = !partial && k1 < KT;
      int c_first = 0, c_last = -1;
      if (head) {
        // clusters after this one whose ranges start inside this tile (an
        // empty range contributes nothing and raises no flag)
        const int64_t tile_end = static_cast<int64_t>(t + 1) * KT;
        c_first = cluster + 1;
        c_last = cluster;
        while (c_last + 1 < clusters && seg.total * (c_last + 1) / clusters < tile_end) ++c_last;
        for (int cc = c_first; cc <= c_last; ++cc) {
          if (seg.total * cc / clusters == seg.total * (cc + 1) / clusters) continue;
          wait_flag(args.sk_flags + 2 * cc + static_cast<int>(rank));
        }
      }
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (warp == 2 && lane == 0) trace_mark(args.trace, 7);
      const uint32_t lane_addr = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
      auto add_one = [&](uint32_t (&r)[32], int c, int cc) {
        const float4* w = reinterpret_cast<const float4*>(
            args.sk_ws + (static_cast<size_t>(2 * cc + rank) * kBM + trow) * BN + c);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 p = w[i];
          r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + p.x);
          r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + p.y);
          r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + p.z);
          r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + p.w);
        }
      };
      auto add_parts = [&](uint32_t (&r)[32], int c) {
        for (int cc = c_first; cc <= c_last; ++cc) {
          if (seg.total * cc / clusters == seg.total * (cc + 1) / clusters) continue;
          const float4* w = reinterpret_cast<const float4*>(
              args.sk_ws + (static_cast<size_t>(2 * cc + rank) * kBM + trow) * BN + c);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 p = w[i];
            r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + p.x);
            r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + p.y);
            r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + p.z);
            r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + p.w);
          }
        }
      };
      uint8_t* stage = staging + (warp - 2) * kStageOut;
      if (partial && args.sk_tma) {  // raw accumulator to this CTA's partial tile
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
          uint32_t r[32];
          tmem_ld32(lane_addr + uint32_t(c), r);
          sk_store_chunk(&args.skmap, stage, lane, r, c, static_cast<int>(blockIdx.x) * kBM + quarter * 32);
        }
        sk_store_done(lane);
      } else if (args.tma_out && !partial) {
        constexpr int kCW = kOutF32 ? 32 : 64;
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += kCW) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
          uint32_t r[kCW / 32][32];
#pragma unroll
          for (int p = 0; p < kCW / 32; ++p) tmem_ld32(lane_addr + uint32_t(c + 32 * p), r[p]);
          if (head) {  // add the later CTAs' partials, in CTA order (deterministic)
            for (int cc = c_first; cc <= c_last; ++cc) {
              if (seg.total * cc / clusters == seg.total * (cc + 1) / clusters) continue;
#pragma unroll
              for (int p = 0; p < kCW / 32; ++p) {
                if (args.sk_tma)
                  sk_add_chunk(&args.skmap, stage, &pbar[warp - 2], pphase, lane, r[p],
                               c + 32 * p, (2 * cc + static_cast<int>(rank)) * kBM + quarter * 32);
                else
                  add_one(r[p], c + 32 * p, cc);
              }
            }
          }
#pragma unroll
          for (int p = 0; p < kCW / 32; ++p) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[p][i]);
            epi_values32<kEpi>(v, row, n0 + c + 32 * p, M, N, args.aux[g], args.ldaux);
            epi_stage32<kOutF32>(stage, lane, p, v);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            for (int j = 0; j < args.fan; ++j)
              tma_store_2d(&args.cmap[g * args.fan + j], stage, n0 + c, m0 + quarter * 32);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (warp == 2) trace_mark(args.trace, 8);
          }
        }
      } else {
#pragma unroll 1
      for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
        uint32_t r[32];
        tmem_ld32(lane_addr + uint32_t(c), r);
        if (partial) {
          float4* w = reinterpret_cast<float4*>(
              args.sk_ws + (static_cast<size_t>(blockIdx.x) * kBM + trow) * BN + c);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            w[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                               __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          continue;
        }
        add_parts(r, c);
        epi_store32<kEpi, kOutF32>(outs, args.fan, ldc, M, N, row, n0 + c, r, args.aux[g],
                                   args.ldaux);
      }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0 && local + 2 < ntiles) remote_arrive(acc_empty_leader + acc * 8);
      if (partial || head) {
        // all 8 epilogue warps of this CTA finished writing / reading
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        if (warp == 2 && lane == 0) {
          if (partial) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(args.sk_flags + blockIdx.x),
                         "r"(1)
                         : "memory");
          } else {
            for (int cc = c_first; cc <= c_last; ++cc) args.sk_flags[2 * cc + rank] = 0;
          }
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (warp == 2 && lane == 0) trace_mark(args.trace, 9);
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) trace_mark(args.trace, 10);
  // peer done with our barriers / TMEM before teardown. Relaxed: no remote
  // operation on shared memory is in flight here (every full-barrier arrive
  // and stage commit was waited on, the unconsumed accumulator-release
  // arrivals are skipped), and a release arrive costs MEMBAR.GPU + ERRBAR
  // (0.5 us per launch, tools/gemm_k_slope.py)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(S::kTmemCols));
    if (lane == 0) trace_mark(args.trace, 11);
  }
}

}  // namespace pair

// ---- host side ---------------------------------------------------------------

// apl_gemm_trace's buffer (nullptr: off).
std::atomic<unsigned long long*> g_trace{nullptr};
std::atomic<int> g_trace_ctas{0};

// APL_DEBUG=1: say which step of a GEMM launch failed (stderr).
bool debug_on() {
  static const bool on = [] {
    const char* e = std::getenv("APL_DEBUG");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}
cudaError_t why(cudaError_t e, const char* what) {
  if (e != cudaSuccess && debug_on())
    std::fprintf(stderr, "apl gemm: %s: %s\n", what, cudaGetErrorString(e));
  return e;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    // by version first (the unversioned query can resolve differently under
    // tools that interpose the driver, e.g. compute-sanitizer)
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess && p != nullptr)
      return reinterpret_cast<EncodeFn>(p);
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// Encoded tensor maps by (pointer, extents, leading dim, box, dtype): a
// training loop reuses its buffers, so most launches skip the driver's
// encode (the host cost that dominated eager small GEMMs). Bounded: cleared
// when it outgrows kMapCache entries.
constexpr size_t kMapCache = 512;
struct MapKey {
  uintptr_t ptr;
  int64_t rows, cols, ld;
  int box_rows, box_cols, f32;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld &&
           box_rows == o.box_rows && box_cols == o.box_cols && f32 == o.f32;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<uintptr_t>()(k.ptr);
    for (int64_t v : {k.rows, k.cols, k.ld, int64_t{k.box_rows}, int64_t{k.box_cols},
                      int64_t{k.f32}})
      h = h * 1000003u ^ std::hash<int64_t>()(v);
    return h;
  }
};
std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

bool cached_map(const MapKey& k, CUtensorMap* map) {
  std::lock_guard<std::mutex> hold(g_map_mu);
  auto it = g_maps.find(k);
  if (it == g_maps.end()) return false;
  *map = it->second;
  return true;
}
void remember_map(const MapKey& k, const CUtensorMap& map) {
  std::lock_guard<std::mutex> hold(g_map_mu);
  if (g_maps.size() >= kMapCache) g_maps.clear();
  g_maps.emplace(k, map);
}

// 2-D bf16 tensor map, 128B swizzle, box = [box_rows][box_cols] (box_cols
// x 2 B = one 128-byte swizzle row).
bool make_map(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, int box_rows,
              int box_cols = kBK) {
  const MapKey key{reinterpret_cast<uintptr_t>(ptr), rows, cols, ld, box_rows, box_cols, 0};
  if (cached_map(key, map)) return true;
  EncodeFn enc = encode_fn();
  if (enc == nullptr) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t elem[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                         strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && debug_on())
    std::fprintf(stderr, "apl gemm: cuTensorMapEncodeTiled(%p, %d x %d, ld %d, box %d x %d) = %d\n",
                 ptr, rows, cols, ld, box_rows, box_cols, static_cast<int>(r));
  if (r == CUDA_SUCCESS) remember_map(key, *map);
  return r == CUDA_SUCCESS;
}

// Output map of the TMA-store epilogue: [rows][cols] of bf16 / fp32 with
// leading dimension ld, box = 32 rows x 128 bytes, 128B swizzle.
bool make_out_map(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, bool f32) {
  const MapKey key{reinterpret_cast<uintptr_t>(ptr), rows, cols, ld, 32, -1, f32 ? 1 : 0};
  if (cached_map(key, map)) return true;
  EncodeFn enc = encode_fn();
  if (enc == nullptr) return false;
  const int elt = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * elt};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / elt), 32};
  const cuuint32_t elem[2] = {1, 1};
  const CUresult r = enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                         2, const_cast<void*>(ptr), dims, strides, box, elem,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS) remember_map(key, *map);
  return r == CUDA_SUCCESS;
}

// APL_GEMM_MC=1: the 4-CTA multicast pair kernel. Off by default: measured
// equal or slower than 2-CTA clusters on every config-5 shape and 8192^3
// (profiles/r02_gemm_sweep_mc.jsonl) -- A operand reads are not the limiter.
bool gemm_mc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_GEMM_MC");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

// APL_GEMM_TMA_OUT=0: per-lane st.global epilogue (A/B).
bool tma_out_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_GEMM_TMA_OUT");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

// APL_GEMM_PDL=0: launch without the programmatic-serialization attribute
// (the kernel's griddepcontrol instructions are then no-ops).
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("APL_GEMM_PDL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

template <typename Kernel>
cudaError_t launch_gemm_kernel(Kernel kernel, int grid, int smem, cudaStream_t stream,
                               const GemmArgs& args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args);
}

// Fill args.cmap for outputs c[0 .. n) when every one can take TMA stores.
void attach_out_maps(GemmArgs& args, int n, bool out_f32) {
  args.tma_out = 0;
  if (!tma_out_enabled() || args.scatter_rows > 0) return;
  const int elt = out_f32 ? 4 : 2;
  if ((static_cast<int64_t>(args.ldc) * elt) % 16) return;
  for (int i = 0; i < n; ++i)
    if ((reinterpret_cast<uintptr_t>(args.c[i]) & 15) ||
        !make_out_map(&args.cmap[i], args.c[i], args.M, args.N, args.ldc, out_f32))
      return;
  args.tma_out = 1;
}

template <int BN, int E, bool F, bool BMN, bool AMN = false>
cudaError_t launch_gemm(const GemmArgs& args, cudaStream_t stream) {
  auto kernel = gemm_bf16_tcgen05<BN, E, F, BMN, AMN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Smem<BN>::kBytes);
    if (e != cudaSuccess) return why(e, "cudaFuncSetAttribute(max dynamic smem)");
    configured = true;
  }
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  const int tiles = ((args.N + BN - 1) / BN) * ((args.M + kBM - 1) / kBM) * args.count;
  const int grid = args.streamk ? (args.sk_units > 0 ? args.sk_units : sms)
                                 : (tiles < sms ? tiles : sms);
  cudaError_t e = launch_gemm_kernel(kernel, grid, Smem<BN>::kBytes, stream, args);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return why(e, "gemm launch");
}

template <int BN, bool BMN>
cudaError_t dispatch(const GemmArgs& args, bool out_f32, int epi, bool a_km,
                     cudaStream_t stream) {
  if (a_km) {  // weight-gradient GEMMs: no activation epilogue
    if (epi != kEpiNone) return cudaErrorInvalidValue;
    return out_f32 ? launch_gemm<BN, kEpiNone, true, BMN, true>(args, stream)
                   : launch_gemm<BN, kEpiNone, false, BMN, true>(args, stream);
  }
  if (epi == kEpiDGelu)
    return out_f32 ? launch_gemm<BN, kEpiDGelu, true, BMN>(args, stream)
                   : launch_gemm<BN, kEpiDGelu, false, BMN>(args, stream);
  if (epi == kEpiGeluSave)
    return out_f32 ? cudaErrorInvalidValue : launch_gemm<BN, kEpiGeluSave, false, BMN>(args, stream);
  if (epi == kEpiGelu)
    return out_f32 ? launch_gemm<BN, kEpiGelu, true, BMN>(args, stream)
                   : launch_gemm<BN, kEpiGelu, false, BMN>(args, stream);
  return out_f32 ? launch_gemm<BN, kEpiNone, true, BMN>(args, stream)
                 : launch_gemm<BN, kEpiNone, false, BMN>(args, stream);
}

// 2-CTA pair kernel launch (cluster dims are compiled into the kernel).
template <int BN, int E, bool F, bool BMN, bool AMN, bool MC>
cudaError_t launch_pair_t(const GemmArgs& args, cudaStream_t stream) {
  auto kernel = pair::gemm_bf16_tcgen05_pair<BN, E, F, BMN, AMN, MC>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         pair::Cfg<BN>::kBytes);
    if (e != cudaSuccess) return why(e, "cudaFuncSetAttribute(max dynamic smem, pair)");
    configured = true;
  }
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  constexpr int kCS = MC ? 4 : 2;
  // co-resident clusters: a persistent grid larger than this runs its last
  // clusters as a second wave (4-CTA clusters do not tile every GPC)
  static const int max_clusters = [&] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kCS * (sms / kCS), 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = pair::Cfg<BN>::kBytes;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = sms / kCS;
    }
    if (debug_on()) std::fprintf(stderr, "apl gemm: %d-CTA clusters co-resident: %d\n", kCS, n);
    return std::min(n, sms / kCS);
  }();
  const int tiles = ((args.N + BN - 1) / BN) *
                    ((args.M + 2 * pair::kBM - 1) / (2 * pair::kBM)) * args.count / (MC ? 2 : 1);
  const int clusters = args.streamk ? (args.sk_units > 0 ? std::min(args.sk_units, max_clusters)
                                                         : max_clusters)
                                     : std::min(tiles, max_clusters);
  unsigned long long* tr = g_trace.load();
  cudaError_t e;
  if (tr != nullptr && kCS * clusters <= g_trace_ctas.load()) {
    GemmArgs traced = args;
    traced.trace = tr;
    traced.trace_ctas = g_trace_ctas.load();
    e = launch_gemm_kernel(kernel, kCS * clusters, pair::Cfg<BN>::kBytes, stream, traced);
  } else {
    e = launch_gemm_kernel(kernel, kCS * clusters, pair::Cfg<BN>::kBytes, stream, args);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return why(e, "pair gemm launch");
}

// args.a_mc: A maps built with 64-row boxes for the multicast cluster kernel.
template <int BN, int E, bool F, bool BMN, bool AMN = false>
cudaError_t launch_pair(const GemmArgs& args, cudaStream_t stream) {
  return args.a_mc ? launch_pair_t<BN, E, F, BMN, AMN, true>(args, stream)
                   : launch_pair_t<BN, E, F, BMN, AMN, false>(args, stream);
}

template <int BN, bool BMN>
cudaError_t dispatch_pair(const GemmArgs& args, bool out_f32, int epi, bool a_km,
                          cudaStream_t stream) {
  if (a_km) {
    if (epi != kEpiNone) return cudaErrorInvalidValue;
    return out_f32 ? launch_pair<BN, kEpiNone, true, BMN, true>(args, stream)
                   : launch_pair<BN, kEpiNone, false, BMN, true>(args, stream);
  }
  switch (epi) {
    case kEpiGelu:
      return out_f32 ? launch_pair<BN, kEpiGelu, true, BMN>(args, stream)
                     : launch_pair<BN, kEpiGelu, false, BMN>(args, stream);
    case kEpiDGelu:
      return out_f32 ? cudaErrorInvalidValue : launch_pair<BN, kEpiDGelu, false, BMN>(args, stream);
    case kEpiGeluSave:
      return out_f32 ? cudaErrorInvalidValue
                     : launch_pair<BN, kEpiGeluSave, false, BMN>(args, stream);
    default:
      return out_f32 ? launch_pair<BN, kEpiNone, true, BMN>(args, stream)
                     : launch_pair<BN, kEpiNone, false, BMN>(args, stream);
  }
}

// Stream-K for single-CTA launches whose tiles fill the SMs badly, e.g.
// per-GPU shards of 8-way strategies (see plan_gemm). Workspace
// (fp32 partial tiles, one per CTA) and flags are kept per stream.
struct StreamKWs {
  float* ws = nullptr;
  int* flags = nullptr;
};

int stream_k_forced() {
  static const int forced = [] {
    const char* e = std::getenv("APL_GEMM_STREAMK");
    return e ? std::atoi(e) : -1;
  }();
  return forced;
}
// APL_GEMM_STREAMK unset: stream-K competes in plan_gemm's cost model only
// when APL_GEMM_SK_AUTO=1 (off until measured; see DESIGN 4.2).
bool stream_k_auto() {
  static const bool on = [] {
    const char* e = std::getenv("APL_GEMM_SK_AUTO");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

std::atomic<int> g_force_pair{-1}, g_force_bn{-1}, g_force_sk{-1};

int sm_count_cached() {
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

// Stream-K workspace: one fp32 128 x 256 partial tile and one flag per CTA,
// kept per stream (partial tiles of one launch are consumed within it).
bool make_out_map(CUtensorMap* map, const void* ptr, int rows, int cols, int ld, bool f32);

bool streamk_attach(GemmArgs& args, cudaStream_t stream, int bn) {
  const int sms = sm_count_cached();
  static std::mutex mu;
  static std::map<cudaStream_t, StreamKWs> pool;
  std::lock_guard<std::mutex> hold(mu);
  StreamKWs& w = pool[stream];
  if (w.ws == nullptr) {
    if (cudaMalloc(&w.ws, static_cast<size_t>(sms) * kBM * 256 * sizeof(float)) != cudaSuccess)
      return false;
    if (cudaMalloc(&w.flags, static_cast<size_t>(sms) * sizeof(int)) != cudaSuccess ||
        cudaMemset(w.flags, 0, static_cast<size_t>(sms) * sizeof(int)) != cudaSuccess)
      return false;
  }
  args.streamk = 1;
  args.sk_ws = w.ws;
  args.sk_flags = w.flags;
  // partial tiles as [CTAs x 128 rows][bn fp32 columns] for the TMA fixup
  args.sk_tma = make_out_map(&args.skmap, w.ws, sms * kBM, bn, bn, true) ? 1 : 0;
  return true;
}

// Which kernel, tile and schedule a GEMM launch uses.
struct GemmPlan {
  bool paired;   // CTA-pair (cta_group::2) kernel, 256-row tiles
  int bn;        // N tile: 128 or 256
  bool streamk;  // stream-K over (tile, k-block) instead of whole tiles
  int split = 0; // > 1: aligned split-K -- stream-K over exactly tiles x split units, so
                 // every unit is one K slice of one tile (one segment, one fixup)
};

// Relative per-SM throughput of each tile shape, calibrated on 8192^3 where
// wave quantisation is negligible, with the TMA-store epilogue and the
// whole-warp MMA issuer and TMA producer (profiles/r02_gemm_sweep_prod.jsonl:
// pair256 1471, pair128 1196, cta256 1176, cta128 903 TFLOP/s). Operand
// fill per MMA cycle sets the order: the 256 x 256 pair tile needs 64 B/clk
// per SM, the others 96-128 B/clk.
double tile_eff(bool paired, int bn) {
  if (paired) return bn == 256 ? 1.0 : 0.81;
  return bn == 256 ? 0.8 : 0.62;
}

// APL_GEMM_SPLITK=<s>: force aligned split-K s (probe); APL_GEMM_SPLIT_AUTO=1
// lets the cost model pick it (off: the per-lane fp32 partial exchange made
// every split slower than whole tiles, profiles/r02_gemm_sweep_split.jsonl).
int split_forced() {
  static const int v = [] {
    const char* e = std::getenv("APL_GEMM_SPLITK");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
bool split_auto() {
  static const bool on = [] {
    const char* e = std::getenv("APL_GEMM_SPLIT_AUTO");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

// Cost model: per-SM work of a tile / its efficiency, times the waves of
// tiles over the resident units (clusters for pairs, CTAs otherwise);
// stream-K spreads the k-blocks evenly and pays ~8% for the fixup; aligned
// split-K s runs tiles x s one-segment units (one wave at most) and pays
// ~10% for its fixup (fp32 partial tiles through L2).
// APL_GEMM_PAIR=0/1, APL_GEMM_BN=128/256, APL_GEMM_STREAMK=0/1 force parts;
// apl_gemm_force_plan's streamk >= 2 forces aligned split-K.
GemmPlan plan_gemm(int M, int N, int K, int count, bool sk_allowed, bool pair_allowed) {
  static const int e_pair = [] {
    const char* e = std::getenv("APL_GEMM_PAIR");
    return e ? std::atoi(e) : -1;
  }();
  static const int e_bn = [] {
    const char* e = std::getenv("APL_GEMM_BN");
    return e ? std::atoi(e) : -1;
  }();
  // apl_gemm_force() overrides (A/B sweeps in one process), then the env
  const int o_pair = g_force_pair.load(), o_bn = g_force_bn.load(), o_sk = g_force_sk.load();
  const int f_pair = o_pair >= 0 ? o_pair : e_pair;
  const int f_bn = o_bn > 0 ? o_bn : e_bn;
  const int f_sk = o_sk >= 0 ? o_sk : stream_k_forced();
  const int sms = sm_count_cached();
  const int kb = (K + kBK - 1) / kBK;
  GemmPlan best{false, 128, false};
  double best_cost = 1e300;
  for (int paired = 0; paired < 2; ++paired) {
    if (paired && !pair_allowed) continue;
    if (f_pair >= 0 && paired != f_pair) continue;
    for (int bn : {128, 256}) {
      if (f_bn > 0 && bn != f_bn) continue;
      const int64_t tm = paired ? 256 : 128;
      const int64_t tiles = ((M + tm - 1) / tm) * ((N + bn - 1) / bn) * count;
      const int units = paired ? sms / 2 : sms;
      const double work = static_cast<double>(tm) * bn / (paired ? 2 : 1) * kb /
                          tile_eff(paired != 0, bn);
      for (int sk = 0; sk < 2; ++sk) {
        if (sk && (!sk_allowed || kb < 4 || tiles * kb < 2 * units)) continue;
        if (f_sk >= 0 && sk != f_sk) continue;
        const double cost = sk ? 1.08 * work * static_cast<double>(tiles) / units
                               : work * static_cast<double>((tiles + units - 1) / units);
        // auto mode keeps stream-K off until it is measured better (r02)
        if (sk && f_sk < 0 && !stream_k_auto()) continue;
        if (cost < best_cost) {
          best_cost = cost;
          best = GemmPlan{paired != 0, bn, sk != 0};
        }
      }
      // aligned split-K: only when the whole tiles leave units idle
      const int fs = o_sk >= 2 ? o_sk : split_forced();
      for (int split : {2, 4}) {
        if (!sk_allowed || kb % split || kb / split < 4 || tiles * split > units) continue;
        if (fs >= 2 ? split != fs : (f_sk >= 0 || fs == 0 || !split_auto())) continue;
        const double cost = 1.1 * work / split;
        if (cost < best_cost || fs >= 2) {
          best_cost = cost;
          best = GemmPlan{paired != 0, bn, true, split};
        }
      }
    }
  }
  return best;
}

}  // namespace

// count equally shaped problems C_i[M,N] = epi(A_i . B_i); A_i given as
// [M,K] (K contiguous) or, with a_km, as row-major [K,M] (M contiguous);
// B_i as Bt [N,K] (b_kn = false, nn.Linear layout) or row-major [K,N]
// (b_kn = true); bf16 in, fp32 accumulate. out_f32 selects the output type;
// epi: 0 none, 1 exact-erf GELU, 2 GELU backward against aux_i (bf16 [M,N],
// leading dimension ldaux, one per output problem). All problems share one
// persistent launch (chunks of kMaxBatch): the CTA-pair kernel (M=256 x
// N=256 tiles) for large forward problems, the single-CTA kernel (128 x BN)
// otherwise.
cudaError_t gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                              int groups, int reduce, int fan, int M, int N, int K, int lda,
                              int ldb, int ldc, bool b_kn, bool out_f32, int epi, bool a_km,
                              const void* const* aux, int ldaux, cudaStream_t stream) {
  if (M <= 0 || N <= 0 || K <= 0 || groups <= 0) return cudaSuccess;
  if (encode_fn() == nullptr)
    return why(cudaErrorSymbolNotFound, "no cuTensorMapEncodeTiled entry point");
  if (reduce < 1 || fan < 1 || reduce > kMaxBatch || fan > kMaxBatch)
    return why(cudaErrorInvalidValue, "reduce / fan outside [1, 8]");
  if ((lda * 2) % 16 || (ldb * 2) % 16)
    return why(cudaErrorInvalidValue, "lda / ldb rows not 16-byte multiples (TMA)");
  if (epi < kEpiNone || epi > kEpiGeluSave || (epi >= kEpiDGelu && aux == nullptr))
    return why(cudaErrorInvalidValue, "bad epilogue / missing aux");
  const int per_launch = std::max(1, std::min(kMaxBatch / reduce, kMaxBatch / fan));
  const GemmPlan plan = plan_gemm(M, N, K, std::min(groups, per_launch),
                                  /*sk_allowed=*/reduce == 1 && fan == 1,
                                  /*pair_allowed=*/!(epi == kEpiDGelu && out_f32));
  const bool paired = plan.paired;
  const int bn = plan.bn;
  // B box rows for the K-major layout: the pair kernel stages half of its
  // N tile per CTA.
  const int b_rows = paired ? bn / 2 : bn;
  // whole-tile pair plans with an even N-tile count run as 4-CTA clusters
  // that multicast A across the two pairs (APL_GEMM_MC=0: 2-CTA clusters)
  const bool mc = paired && !plan.streamk && ((N + bn - 1) / bn) % 2 == 0 && gemm_mc_enabled();
  for (int first = 0; first < groups; first += per_launch) {
    GemmArgs args;
    std::memset(&args, 0, sizeof(args));
    args.count = std::min(per_launch, groups - first);
    args.reduce = reduce;
    args.fan = fan;
    args.M = M;
    args.N = N;
    args.K = K;
    args.ldc = ldc;
    args.ldaux = ldaux;
    for (int i = 0; i < args.count * reduce; ++i) {
      const void* a = A[first * reduce + i];
      const void* b = B[first * reduce + i];
      if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(b) & 15))
        return why(cudaErrorInvalidValue, "operand base not 16-byte aligned (TMA)");
      const bool oka = a_km ? make_map(&args.a[i], a, K, M, lda, kBK, 64)
                            : make_map(&args.a[i], a, M, K, lda, mc ? kBM / 2 : kBM);
      const bool okb = b_kn ? make_map(&args.b[i], b, K, N, ldb, kBK, 64)
                            : make_map(&args.b[i], b, N, K, ldb, b_rows);
      if (!oka || !okb) return why(cudaErrorInvalidValue, "tensor map encode");
    }
    for (int i = 0; i < args.count * fan; ++i) args.c[i] = C[first * fan + i];
    attach_out_maps(args, args.count * fan, out_f32);
    args.a_mc = mc ? 1 : 0;
    if (epi >= kEpiDGelu)
      for (int i = 0; i < args.count; ++i) args.aux[i] = aux[first + i];
    if (plan.streamk && !streamk_attach(args, stream, bn)) return cudaErrorMemoryAllocation;
    if (plan.split > 1) {
      const int64_t tm = paired ? 256 : 128;
      args.sk_units = static_cast<int>(((M + tm - 1) / tm) * ((N + bn - 1) / bn) *
                                       args.count * plan.split);
    }
    cudaError_t e;
    if (paired && bn == 256)
      e = b_kn ? dispatch_pair<256, true>(args, out_f32, epi, a_km, stream)
               : dispatch_pair<256, false>(args, out_f32, epi, a_km, stream);
    else if (paired)
      e = b_kn ? dispatch_pair<128, true>(args, out_f32, epi, a_km, stream)
               : dispatch_pair<128, false>(args, out_f32, epi, a_km, stream);
    else if (b_kn)
      e = bn == 256 ? dispatch<256, true>(args, out_f32, epi, a_km, stream)
                    : dispatch<128, true>(args, out_f32, epi, a_km, stream);
    else
      e = bn == 256 ? dispatch<256, false>(args, out_f32, epi, a_km, stream)
                    : dispatch<128, false>(args, out_f32, epi, a_km, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                              int groups, int reduce, int fan, int M, int N, int K, int lda,
                              int ldb, int ldc, bool b_kn, bool out_f32, bool gelu,
                              cudaStream_t stream) {
  return gemm_bf16_grouped(A, B, C, groups, reduce, fan, M, N, K, lda, ldb, ldc, b_kn, out_f32,
                           gelu ? kEpiGelu : kEpiNone, false, nullptr, 0, stream);
}

// Fused GEMM + reduce-scatter send: C = A . B (one problem) with row block
// q (M / owners rows) of the fp32 partial written to owner_slabs[q] (the
// owner's staging slab reserved for this rank; peer-mapped pointers on a
// peer mesh). M / owners must be a multiple of the 128-row tile.
cudaError_t gemm_bf16_scatter(const void* A, const void* B, void* const* owner_slabs, int owners,
                              int M, int N, int K, int lda, int ldb, bool b_kn,
                              cudaStream_t stream) {
  if (owners < 1 || owners > kMaxBatch || M % owners || (M / owners) % kBM)
    return cudaErrorInvalidValue;
  if ((lda * 2) % 16 || (ldb * 2) % 16) return cudaErrorInvalidValue;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15))
    return cudaErrorInvalidValue;
  GemmArgs args;
  std::memset(&args, 0, sizeof(args));
  args.count = 1;
  args.reduce = 1;
  args.fan = 1;
  args.M = M;
  args.N = N;
  args.K = K;
  args.ldc = N;
  args.scatter_rows = M / owners;
  const int bn = (N >= 256 && N % 256 == 0) ? 256 : 128;
  if (!make_map(&args.a[0], A, M, K, lda, kBM)) return cudaErrorInvalidValue;
  const bool okb = b_kn ? make_map(&args.b[0], B, K, N, ldb, kBK, 64)
                        : make_map(&args.b[0], B, N, K, ldb, bn);
  if (!okb) return cudaErrorInvalidValue;
  for (int q = 0; q < owners; ++q) args.c[q] = owner_slabs[q];
  if (b_kn)
    return bn == 256 ? dispatch<256, true>(args, true, kEpiNone, false, stream)
                     : dispatch<128, true>(args, true, kEpiNone, false, stream);
  return bn == 256 ? dispatch<256, false>(args, true, kEpiNone, false, stream)
                   : dispatch<128, false>(args, true, kEpiNone, false, stream);
}

cudaError_t gemm_bf16_batched(const void* const* A, const void* const* B, void* const* C,
                              int count, int M, int N, int K, int lda, int ldb, int ldc,
                              bool b_kn, bool out_f32, bool gelu, cudaStream_t stream) {
  return gemm_bf16_grouped(A, B, C, count, 1, 1, M, N, K, lda, ldb, ldc, b_kn, out_f32, gelu,
                           stream);
}

cudaError_t gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                      int ldb, int ldc, bool b_kn, bool out_f32, bool gelu, cudaStream_t stream) {
  return gemm_bf16_batched(&A, &B, &C, 1, M, N, K, lda, ldb, ldc, b_kn, out_f32, gelu, stream);
}

// Force parts of the GEMM plan (-1: automatic): the CTA pair kernel, the N
// tile, stream-K. For A/B measurements (tools/gemm_bench.py --sweep).
// Diagnostics: CTA-pair GEMM launches record per-CTA phase timestamps into
// `buf` (kTraceSlots u64 per CTA; nullptr turns it off). A launch whose grid
// has more CTAs than `bytes` holds runs untraced.
void gemm_trace(void* buf, size_t bytes) {
  g_trace_ctas.store(buf ? static_cast<int>(bytes / (kTraceSlots * sizeof(unsigned long long))) : 0);
  g_trace.store(static_cast<unsigned long long*>(buf));
}

void gemm_force_plan(int pair, int bn, int streamk) {
  g_force_pair.store(pair);
  g_force_bn.store(bn);
  g_force_sk.store(streamk);
}

cudaError_t gemm_bf16_tn(const void* A, const void* Bt, void* C, int M, int N, int K, int lda,
                         int ldb, int ldc, bool out_f32, bool gelu, cudaStream_t stream) {
  return gemm_bf16(A, Bt, C, M, N, K, lda, ldb, ldc, false, out_f32, gelu, stream);
}

}  // namespace apl
