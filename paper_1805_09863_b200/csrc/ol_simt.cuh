// ol_simt.cuh — fp32 fused output layer on the CUDA cores.
//
// The fp32 configuration (BASELINE.json cfg "tiny") needs true fp32 products:
// TF32 inputs miss the 1e-4 relative cost tolerance.
// Same schedule, same partial records and the same per-row epilogue
// (RowState::chunk32) as the tcgen05 kernel: thread = hypothesis row, 32
// logits per chunk accumulated in registers in ascending h (fixed order).
#pragma once
#include "epilogue.cuh"

namespace amun {

struct SimtParams {
  int N, V_local, v_offset, H;
  Schedule sch;
  const float* __restrict__ X;   // [N][H]
  const float* __restrict__ W;   // [V_local][H]
  const float* __restrict__ bias;
  float* __restrict__ part;
  int stride, k_max;
  float* __restrict__ logits;    // MODE 1
};

constexpr int SIMT_KC = 32;

template <int KB, int MODE>
__global__ void __launch_bounds__(128) ol_simt_kernel(const SimtParams p) {
  __shared__ float xs[128][SIMT_KC + 1];
  __shared__ __align__(16) float ws[32][SIMT_KC];
  __shared__ __align__(128) float xsc[128 * 32];
  const int tid = threadIdx.x;
  RowState<KB> st;
  st.reset();
  const long long start = (long long)blockIdx.x * p.sch.C;
  const long long stop = min(start + p.sch.C, p.sch.total);
  TileIter it{start, stop, p.sch};
  int mt, v0, width;
  bool last;
  while (it.next(mt, v0, width, last)) {
    const int row = mt * 128 + tid;
    const int limit = min(width, p.V_local - v0);
    for (int c = 0; c < width; c += 32) {
      float acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.f;
      for (int k0 = 0; k0 < p.H; k0 += SIMT_KC) {
        __syncthreads();
        for (int e = tid; e < 128 * SIMT_KC; e += 128) {
          const int rr = e / SIMT_KC, kk = e % SIMT_KC;
          const int gr = mt * 128 + rr, gk = k0 + kk;
          xs[rr][kk] = (gr < p.N && gk < p.H) ? p.X[(long long)gr * p.H + gk] : 0.f;
        }
        for (int e = tid; e < 32 * SIMT_KC; e += 128) {
          const int jj = e / SIMT_KC, kk = e % SIMT_KC;
          const int gv = v0 + c + jj, gk = k0 + kk;
          ws[jj][kk] = (c + jj < limit && gk < p.H) ? p.W[(long long)gv * p.H + gk] : 0.f;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < SIMT_KC; ++kk) {
          const float xv = xs[tid][kk];
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = fmaf(xv, ws[j][kk], acc[j]);
        }
      }
      const int nv = limit - c;
      float x[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = (j < nv) ? acc[j] + __ldg(p.bias + v0 + c + j) : kNegInf;
      if constexpr (MODE == 1) {
        if (row < p.N) {
          float* out = p.logits + (long long)row * p.V_local + v0 + c;
          for (int j = 0; j < 32 && j < nv; ++j) out[j] = x[j];
        }
      } else {
        st.chunk32(x, p.v_offset + v0 + c, xsc + tid * 32, tid & 7);
      }
    }
    if (last) {
      if constexpr (MODE == 0) {
        if (row < p.N) {
          const long long slot = (long long)blockIdx.x + mt;
          st.emit(p.part + (slot * 128 + tid) * p.stride, p.k_max);
        }
      }
      st.reset();
    }
  }
}

}  // namespace amun
