// gemm_skinny.cu — APT W_p x A_q product for decode-sized token counts (M <= 16) with legacy
// mma.sync.m16n8k32 u8 tensor-core instructions fed straight from registers.
//
// Why: the tcgen05 decode tile is paced by the MMA reading its 4 KB weight operand
// per 128 x 16 x 32 instruction out of TMEM and by its mbarrier / TMEM / cluster round trips; the
// SIMT GEMV (gemv.cu) showed that a kernel with no on-chip staging at all — one HBM round trip
// plus arithmetic — is 1.3-2.2x faster at M <= 2.  This kernel keeps that structure and moves the
// multiply-accumulate onto the tensor cores so it scales to 16 tokens:
//   * CTA = 16 weight rows (the MMA M side) x all tokens (BN = 8 NT <= 16) x the whole K range; its
//     NW warps split K (iterations of 256 elements) and meet in shared memory;
//   * lane (g, t) = (lane / 4, lane % 4) loads words 2t and 2t+1 of each 256-element iteration of rows
//     g and g+8 for every plane — in the tile-major layout (APT_PACK_TILED) a warp's loads are two
//     256-byte contiguous runs per plane — requested for a batch of iterations ahead of use, the
//     first batch before griddepcontrol.wait;
//   * rebuild8() (the shift half of the shift-add recovery, the same u8 digits as every other
//     kernel) turns a word into 8 digit registers; register 2s / 2s+1 of word 2t+grp are the A
//     fragment's k-slots [4t, 4t+4) / [16+4t, 16+4t+4) of K-step s of group grp, and the token
//     operand takes the same registers of the same word from the activation digit view, so both
//     operands agree on K;
//   * 8 mma.sync per iteration and 8-token tile accumulate u8 x u8 into s32 (the add half);
//   * epilogue: the warps' partial tiles are summed in shared memory and every output goes through
//     epilogue_store_v (rank-1 correction, fp16 scale, row or column layout).
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

constexpr int kSkRows = 16;  // weight rows per CTA (MMA M)

template <int NW>
struct SkShape {
  static constexpr int kMinBlocks = NW >= 16 ? 1 : NW >= 8 ? 3 : 6;
};

__device__ __forceinline__ void mma_u8_16816(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int WB, int NT, int NW>
__global__ void __launch_bounds__(32 * NW, SkShape<NW>::kMinBlocks) gemm_skinny_kernel(GemvArgs p) {
  constexpr int BN = 8 * NT;
  // iterations whose weight loads are in flight together (double-buffered)
#ifdef APT_SK_BATCH
  constexpr int kBatch = APT_SK_BATCH;
#else
  constexpr int kBatch = WB <= 2 ? 2 : 1;
#endif
  // independent accumulator chains per 8-token tile (consecutive mma.sync into one accumulator
  // serialise on the MMA latency)
#ifdef APT_SK_ACC
  constexpr int kAcc = APT_SK_ACC;
#else
  constexpr int kAcc = 1;
#endif
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int r0 = blockIdx.x * kSkRows;
  const int m0 = blockIdx.y * BN;
  const int ra = min(r0 + g, p.e.N - 1), rb = min(r0 + g + 8, p.e.N - 1);
  const int n_it = p.k_words >> 3;  // 256-element iterations
  const int i0 = (warp * n_it) / NW, i1 = ((warp + 1) * n_it) / NW;
  const int kw8 = p.k_words >> 3;
  auto wptr = [&](int r, int it, int i) -> const uint2* {
    const uint32_t* b = p.wp + (int64_t)i * p.w_pstride;
    return reinterpret_cast<const uint2*>(
        p.w_tiled ? b + ((int64_t)(r >> 7) * kw8 + it) * 1024 + (t >> 1) * 512 + (r & 127) * 4 + (t & 1) * 2
                  : b + (int64_t)r * p.k_words + it * 8 + 2 * t);
  };
  uint2 va[kBatch][WB], vb[kBatch][WB];
  auto load_batch = [&](int ib) {
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
      if (ib + b < i1) {
#pragma unroll
        for (int i = 0; i < WB; ++i) {
          va[b][i] = __ldg(wptr(ra, ib + b, i));
          vb[b][i] = __ldg(wptr(rb, ib + b, i));
        }
      }
  };
  int c[NT][kAcc][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int q = 0; q < kAcc; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[nt][q][j] = 0;
  load_batch(i0);
  pdl_wait();  // activation digits, row sums and scales may come from the previous kernel
  // this lane's token rows (one per 8-token tile), clamped: columns >= M are never stored
  const uint8_t* tok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) tok[nt] = p.adig + (int64_t)min(m0 + nt * 8 + g, p.e.M - 1) * p.k_words * 32;
  for (int ib = i0; ib < i1; ib += kBatch) {
    uint2 ca[kBatch][WB], cb[kBatch][WB];
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
#pragma unroll
      for (int i = 0; i < WB; ++i) {
        ca[b][i] = va[b][i];
        cb[b][i] = vb[b][i];
      }
    if (ib + kBatch < i1) load_batch(ib + kBatch);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int it = ib + b;
      if (it >= i1) break;
#pragma unroll
      for (int grp = 0; grp < 2; ++grp) {
        uint32_t wa[WB], wb[WB], oa[8], ob[8];
#pragma unroll
        for (int i = 0; i < WB; ++i) {
          wa[i] = grp ? ca[b][i].y : ca[b][i].x;
          wb[i] = grp ? cb[b][i].y : cb[b][i].x;
        }
        rebuild8<WB>(wa, oa);
        rebuild8<WB>(wb, ob);
        const int word = it * 8 + 2 * t + grp;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint4* tp = reinterpret_cast<const uint4*>(tok[nt] + (int64_t)word * 32);
          const uint4 d0 = __ldg(tp), d1 = __ldg(tp + 1);
          const uint32_t d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
          for (int s = 0; s < 4; ++s)
            mma_u8_16816(c[nt][(grp * 4 + s) % kAcc], oa[2 * s], ob[2 * s], oa[2 * s + 1], ob[2 * s + 1], d[2 * s],
                         d[2 * s + 1]);
        }
      }
    }
  }
  // the NW partial 16 x BN tiles meet in shared memory
  __shared__ int32_t red[NW][kSkRows][BN];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int q = 1; q < kAcc; ++q)
#pragma unroll
      for (int j = 0; j < 4; ++j) c[nt][0][j] += c[nt][q][j];
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    red[warp][g][nt * 8 + 2 * t] = c[nt][0][0];
    red[warp][g][nt * 8 + 2 * t + 1] = c[nt][0][1];
    red[warp][g + 8][nt * 8 + 2 * t] = c[nt][0][2];
    red[warp][g + 8][nt * 8 + 2 * t + 1] = c[nt][0][3];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < kSkRows * BN; o += 32 * NW) {
    const int row = o / BN, col = o % BN;
    const int n = r0 + row, m = m0 + col;
    if (n < p.e.N && m < p.e.M) {
      uint32_t U = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) U += (uint32_t)red[w][row][col];
      epilogue_store_v(p.e, m, n, U, __ldg(p.e.a_rowsum + m), __ldg(p.e.w_rowsum + n),
                       p.e.kind == 2 ? __ldg(p.e.w_scale + n) : 0.f,
                       (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f);
    }
  }
}

template <int WB, int NW>
static cudaError_t launch_sk2(const GemvArgs& p, int bn, cudaStream_t stream) {
  const dim3 block(32 * NW);
  if (bn == 8) {
    const dim3 grid((p.e.N + kSkRows - 1) / kSkRows, (p.e.M + 7) / 8);
    return launch_pdl(gemm_skinny_kernel<WB, 1, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
  }
  const dim3 grid((p.e.N + kSkRows - 1) / kSkRows, (p.e.M + 15) / 16);
  return launch_pdl(gemm_skinny_kernel<WB, 2, NW>, grid, block, 0, stream, dim3(1, 1, 1), p);
}

template <int WB>
static cudaError_t launch_sk1(const GemvArgs& p, int bn, int warps, cudaStream_t stream) {
  switch (warps) {
    case 4: return launch_sk2<WB, 4>(p, bn, stream);
    case 16: return launch_sk2<WB, 16>(p, bn, stream);
    default: return launch_sk2<WB, 8>(p, bn, stream);
  }
}

cudaError_t launch_gemm_skinny(const GemvArgs& p, int wbits, int bn, int warps, cudaStream_t stream) {
  switch (wbits) {
    case 1: return launch_sk1<1>(p, bn, warps, stream);
    case 2: return launch_sk1<2>(p, bn, warps, stream);
    case 3: return launch_sk1<3>(p, bn, warps, stream);
    case 4: return launch_sk1<4>(p, bn, warps, stream);
    case 5: return launch_sk1<5>(p, bn, warps, stream);
    case 6: return launch_sk1<6>(p, bn, warps, stream);
    case 7: return launch_sk1<7>(p, bn, warps, stream);
    default: return launch_sk1<8>(p, bn, warps, stream);
  }
}

}  // namespace apt
