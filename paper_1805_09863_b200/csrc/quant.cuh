// quant.cuh — per-row FP8 (E4M3) quantisation for the e4m3 output layer
// (the modern analogue of the paper's 16-bit storage,
// P:264-268). Row r: scale_r = max_h |x_rh| / 448 (1 for an all-zero row),
// code_rh = RNE-to-E4M3(x_rh / scale_r) saturating at +-448; IEEE fp32
// division (no fast-math), so the codes match oracle.quantize_rows_e4m3 bit
// for bit. One CTA per row (grid-stride), 256 threads.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

namespace amun {

constexpr int QZ_THREADS = 256;

template <bool BF16>
__global__ void __launch_bounds__(QZ_THREADS) quantize_e4m3_kernel(const void* __restrict__ src,
                                                                   int R, int H,
                                                                   uint8_t* __restrict__ dst,
                                                                   float* __restrict__ scale) {
  __shared__ float red[QZ_THREADS / 32];
  // the fused output-layer kernel that reads these codes is launched with
  // programmatic stream serialization: let it start its prologue now (it
  // waits for this grid's completion before any global access)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x;
  for (int r = blockIdx.x; r < R; r += gridDim.x) {
    auto at = [&](int h) -> float {
      if constexpr (BF16)
        return __bfloat162float(static_cast<const __nv_bfloat16*>(src)[(long long)r * H + h]);
      else
        return static_cast<const float*>(src)[(long long)r * H + h];
    };
    float amax = 0.f;
    for (int h = tid; h < H; h += QZ_THREADS) amax = fmaxf(amax, fabsf(at(h)));
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((tid & 31) == 0) red[tid >> 5] = amax;
    __syncthreads();
    amax = red[0];
#pragma unroll
    for (int w = 1; w < QZ_THREADS / 32; ++w) amax = fmaxf(amax, red[w]);
    __syncthreads();   // red[] reused by the next row
    const float sc = amax > 0.f ? __fdiv_rn(amax, 448.f) : 1.f;
    if (tid == 0) scale[r] = sc;
    uint16_t* d2 = reinterpret_cast<uint16_t*>(dst + (long long)r * H);
    for (int h = 2 * tid; h < H; h += 2 * QZ_THREADS) {
      const float lo = __fdiv_rn(at(h), sc), hi = __fdiv_rn(at(h + 1), sc);
      uint16_t q;
      // e4m3x2: the first source lands in the upper byte
      asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(q) : "f"(hi), "f"(lo));
      d2[h >> 1] = q;
    }
  }
}

// MXFP4 quantisation (amun_quantize_mxfp4; OCP MX v1.0, oracle
// quantize_rows_mxfp4): one warp per (row, 128-element K block), lane l
// converts elements 4l..4l+3; the 8 lanes of a 32-element MX block reduce
// its max |x|. Shared exponent e = floor(log2 amax) - 2 (the biased fp32
// exponent of amax minus 2 is the E8M0 code; 127 for an all-zero block;
// clamped to [0, 254]); codes = RNE-to-E2M1(x * 2^-e), saturating, two per
// byte, the lower element in the low nibble. Scales go to the
// [kblock][row / 128][512-byte atom] layout the fused kernel copies to TMEM
// (amun.h). Rows R..R_pad-1 of the last 128-row atom get code 127 (their W
// rows read as zero).
template <bool BF16>
__global__ void __launch_bounds__(QZ_THREADS) quantize_mxfp4_kernel(const void* __restrict__ src,
                                                                    int R, int H,
                                                                    uint8_t* __restrict__ codes,
                                                                    uint8_t* __restrict__ sf) {
  const int lane = threadIdx.x & 31;
  const int KT = H / 128;
  const long long Rp = (R + 127LL) / 128 * 128;
  const long long tasks = Rp * KT;
  const long long nwarps = (long long)gridDim.x * (QZ_THREADS / 32);
  for (long long t = blockIdx.x * (long long)(QZ_THREADS / 32) + (threadIdx.x >> 5); t < tasks;
       t += nwarps) {
    const long long r = t / KT;
    const int kt = (int)(t - r * KT);
    const int kb = lane >> 3;
    float q[4] = {0.f, 0.f, 0.f, 0.f};
    float amax = 0.f;
    if (r < R) {
      const long long base = r * H + kt * 128 + 4 * lane;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (BF16)
          q[j] = __bfloat162float(static_cast<const __nv_bfloat16*>(src)[base + j]);
        else
          q[j] = static_cast<const float*>(src)[base + j];
        amax = fmaxf(amax, fabsf(q[j]));
      }
    }
#pragma unroll
    for (int o = 4; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    int code = 127;
    if (amax > 0.f) code = min(max((int)((__float_as_uint(amax) >> 23) & 0xffu) - 2, 0), 254);
    if (r < R) {
      uint16_t out;
      const int sh = 127 - code;   // x * 2^-e, exact (a power of two)
      asm("{\n\t.reg .b8 b0, b1;\n\t"
          "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
          "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
          "mov.b16 %0, {b0, b1};\n\t}"
          : "=h"(out)
          : "f"(ldexpf(q[0], sh)), "f"(ldexpf(q[1], sh)), "f"(ldexpf(q[2], sh)),
            "f"(ldexpf(q[3], sh)));
      reinterpret_cast<uint16_t*>(codes + r * (H / 2) + kt * 64)[lane] = out;
    }
    if ((lane & 7) == 0) {
      const long long m = r & 127;
      sf[((long long)kt * (Rp >> 7) + (r >> 7)) * 512 + 16 * (m & 31) + 4 * (m >> 5) + kb] =
          (uint8_t)code;
    }
  }
}

// 3xTF32 split (amun_split_tf32x3): hi = tf32(x), lo = tf32(x - hi); row r
// of dst = role 0: [hi | hi | lo], role 1: [hi | lo | hi].
__global__ void split_tf32x3_kernel(const float* __restrict__ src, long long n, int H, int role,
                                    float* __restrict__ dst) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / H;
    const int h = (int)(i - r * H);
    const float x = src[i];
    uint32_t hb, lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
    const float hi = __uint_as_float(hb);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(x - hi));
    const float lo = __uint_as_float(lb);
    float* row = dst + r * 3LL * H;
    row[h] = hi;
    row[H + h] = role == 0 ? hi : lo;
    row[2 * H + h] = role == 0 ? lo : hi;
  }
}

}  // namespace amun
