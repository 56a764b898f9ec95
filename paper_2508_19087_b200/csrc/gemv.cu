// gemv.cu — APT W_p x A_q product for a handful of tokens (M <= 4) on the integer ALUs.
//
// With M = 1 the tensor-core path is bound by latency and by the MMA reading its 4 KB weight
// operand per 128 x 16 x 32 instruction from TMEM, not by HBM.  SURVEY §8 a9 names
// the SIMT dot-product GEMV (SPEC gemv_ap) as the legal alternative at M = 1 "picked by
// measurement"; this is it, B200-style:
//   * one CTA = 32 weight rows x the whole K range, NW = 8 or 16 warps; lane = weight row, warp w =
//     K steps [w*ns/NW, (w+1)*ns/NW) (ns = Kpad/128).  The weight planes are read straight from HBM with 16-byte
//     vector loads — in the tile-major layout (APT_PACK_TILED) the 32 lanes of a warp read 512
//     contiguous bytes per plane and step — issued for a batch of steps before any is used, and the
//     first batch before griddepcontrol.wait (weights never depend on the previous kernel);
//   * the shift half of the shift-add recovery is the same rebuild8() operand rebuild as the
//     tensor-core kernel (u8 offset digits, K permuted inside each 32-element word identically for
//     both operands); the add half is __dp4a on four digit pairs (u8 x u8 -> u32) against the
//     activation digit view (apt_packed.digits, read once per warp as broadcast vector loads);
//   * the 8 warps' partial sums meet in shared memory; warp 0 applies the rank-1 correction and the
//     scale epilogue (epilogue_store_v, common.cuh: signed / bipolar int32 or fp16, row or column).
// No tensor memory, no cluster, no mbarrier: a launch is one HBM round trip plus the arithmetic.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

constexpr int kGvRows = 32;  // weight rows per CTA (= lanes)

// NW warps split K inside the CTA.  Measured on B200 (tools/gemv_ab.py): the grid must cover the
// machine with short CTAs — 16 warps (one CTA per SM) when the N/32 row tiles do not fill 148 SMs,
// else 8 warps at three CTAs per SM (<= 85 registers).
template <int NW>
struct GvShape {
  static constexpr int kMinBlocks = NW >= 16 ? 1 : 3;
};

template <int WB, int MT, int NW>
__global__ void __launch_bounds__(kGvRows * NW, GvShape<NW>::kMinBlocks) gemv_kernel(GemvArgs p) {
  constexpr int kGvWarps = NW;
  // K steps whose weight loads are in flight together (double-buffered: 2 x kGvBatch x WB x 16 B per
  // lane); with 8 warps at K = 4096 a warp's whole K range is one batch at W <= 2 (one HBM round
  // trip), measured 7-11% faster on 11008 x 4096 than batches of 2 / 1
  constexpr int kGvBatch = WB <= 2 ? 4 : WB <= 4 ? 2 : 1;
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.x * kGvRows + lane;           // weight row of this lane
  const int rr = r < p.e.N ? r : p.e.N - 1;            // clamped (row layout has no pad rows)
  const int ns = p.k_words / 4;                        // 128-element K steps
  const int s0 = (warp * ns) / kGvWarps, s1 = ((warp + 1) * ns) / kGvWarps;
  const int kw8 = p.k_words >> 3;
  auto wptr = [&](int s, int i) -> const uint4* {
    const uint32_t* b = p.wp + (int64_t)i * p.w_pstride;
    return reinterpret_cast<const uint4*>(
        p.w_tiled ? b + ((int64_t)(rr >> 7) * kw8 + (s >> 1)) * 1024 + (s & 1) * 512 + (rr & 127) * 4
                  : b + (int64_t)rr * p.k_words + s * 4);
  };
  uint32_t U[MT], U2[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) U[m] = U2[m] = 0u;
  uint4 v[kGvBatch][WB];
  auto load_batch = [&](int sb) {
#pragma unroll
    for (int b = 0; b < kGvBatch; ++b)
      if (sb + b < s1) {
#pragma unroll
        for (int i = 0; i < WB; ++i) v[b][i] = __ldg(wptr(sb + b, i));
      }
  };
  load_batch(s0);
  pdl_wait();  // the activation digits / row sums / scales may come from the previous kernel
  for (int sb = s0; sb < s1; sb += kGvBatch) {
    uint4 cur[kGvBatch][WB];
#pragma unroll
    for (int b = 0; b < kGvBatch; ++b)
#pragma unroll
      for (int i = 0; i < WB; ++i) cur[b][i] = v[b][i];
    if (sb + kGvBatch < s1) load_batch(sb + kGvBatch);
#pragma unroll
    for (int b = 0; b < kGvBatch; ++b) {
      if (sb + b >= s1) break;
      const int s = sb + b;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t w[WB], o[8];
#pragma unroll
        for (int i = 0; i < WB; ++i) w[i] = q == 0 ? cur[b][i].x : q == 1 ? cur[b][i].y : q == 2 ? cur[b][i].z : cur[b][i].w;
        rebuild8<WB>(w, o);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          // the activation word's 32 digits (same for every lane: one broadcast transaction)
          const uint4* ad = reinterpret_cast<const uint4*>(p.adig + (int64_t)m * p.k_words * 32 + (s * 4 + q) * 32);
          const uint4 a0 = __ldg(ad), a1 = __ldg(ad + 1);
          // two independent dp4a chains (U and U2) halve the dependent-latency chain per word
          uint32_t acc = U[m], acc2 = U2[m];
          acc = __dp4a(o[0], a0.x, acc);
          acc2 = __dp4a(o[1], a0.y, acc2);
          acc = __dp4a(o[2], a0.z, acc);
          acc2 = __dp4a(o[3], a0.w, acc2);
          acc = __dp4a(o[4], a1.x, acc);
          acc2 = __dp4a(o[5], a1.y, acc2);
          acc = __dp4a(o[6], a1.z, acc);
          acc2 = __dp4a(o[7], a1.w, acc2);
          U[m] = acc;
          U2[m] = acc2;
        }
      }
    }
  }
  __shared__ uint32_t red[kGvWarps][MT][kGvRows];
#pragma unroll
  for (int m = 0; m < MT; ++m) red[warp][m][lane] = U[m] + U2[m];
  __syncthreads();
  if (warp == 0 && r < p.e.N) {
    const int32_t rw = __ldg(p.e.w_rowsum + r);
    const float wsc = p.e.kind == 2 ? __ldg(p.e.w_scale + r) : 0.f;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (m >= p.e.M) break;
      uint32_t t = 0;
#pragma unroll
      for (int w = 0; w < kGvWarps; ++w) t += red[w][m][lane];
      epilogue_store_v(p.e, m, r, t, __ldg(p.e.a_rowsum + m), rw, wsc,
                       (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f);
    }
  }
}

template <int WB, int NW>
static cudaError_t launch_gemv2(const GemvArgs& p, cudaStream_t stream) {
  const dim3 grid((p.e.N + kGvRows - 1) / kGvRows), block(kGvRows * NW);
  switch (p.e.M) {
    case 1: return launch_pdl(gemv_kernel<WB, 1, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 2: return launch_pdl(gemv_kernel<WB, 2, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 3: return launch_pdl(gemv_kernel<WB, 3, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
    case 4: return launch_pdl(gemv_kernel<WB, 4, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
    default: return cudaErrorInvalidValue;
  }
}

template <int WB>
static cudaError_t launch_gemv1(const GemvArgs& p, int warps, cudaStream_t stream) {
  return warps == 16 ? launch_gemv2<WB, 16>(p, stream) : launch_gemv2<WB, 8>(p, stream);
}

cudaError_t launch_gemv(const GemvArgs& p, int wbits, int warps, cudaStream_t stream) {
  switch (wbits) {
    case 1: return launch_gemv1<1>(p, warps, stream);
    case 2: return launch_gemv1<2>(p, warps, stream);
    case 3: return launch_gemv1<3>(p, warps, stream);
    case 4: return launch_gemv1<4>(p, warps, stream);
    case 5: return launch_gemv1<5>(p, warps, stream);
    case 6: return launch_gemv1<6>(p, warps, stream);
    case 7: return launch_gemv1<7>(p, warps, stream);
    default: return launch_gemv1<8>(p, warps, stream);
  }
}

}  // namespace apt
