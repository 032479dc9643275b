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
