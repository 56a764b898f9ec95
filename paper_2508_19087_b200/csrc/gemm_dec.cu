// gemm_dec.cu — APT W_p x A_q product for decode token counts (M <= 16): weights streamed as the
// B operand of mma.sync.m16n8k32 u8, the (at most 16) tokens held in registers as the A operand.
//
// Why this shape (measured on B200, tools/probe/mma_rates.cu, profiles/r2_mma_rates.jsonl):
//   * decode is bound by streaming the packed weights; 6.55 TB/s over 148 SMs is ~22 B
//     per SM clock, i.e. 180 / 90 / 60 / 45 weight elements per clock at W1 / W2 / W3 / W4;
//   * tcgen05.mma kind::i8 M=128 with N <= 64 takes ~46 clocks whatever N (it is paced by reading the
//     4 KB A tile), i.e. 90 weight elements per clock; legacy mma.sync m16n8k32 u8 runs at 2048 MAC
//     per clock per SM = one instruction per 2 clocks, and with the weights on its N side (8 rows x 32
//     K = 256 elements per instruction, all 16 token slots useful) that is 128 elements per clock —
//     with no TMEM allocation, mbarrier, cluster or shared-memory operand staging per launch;
//   * the integer ALU pipe issues 64 LOP3 per clock per SM, so the plane -> digit rebuild (the shift
//     half of the shift-add recovery) is the other limit; 1- and 2-bit weights use
//     rebuild_hi (common.cuh), whose shifts run on the FMA pipe.
//
// Work decomposition: a CTA = NW warps = 32 weight rows (four 8-row MMA groups) x one K range
// (gridDim.z = S ranges, normally S = 1); its warps split the range's 256-element blocks and meet in
// shared memory.  Per block each lane (g, t) = (lane / 4, lane % 4) rebuilds words 2t, 2t+1 of row g of
// each group; the same (word, register) pairs of the activation digit view (tokens g and g + 8) form the
// A fragment, so both operands agree on K; 8 MMAs per group accumulate u8 x u8 into s32.  Token
// fragments are loaded straight from the digit view (L2) one block ahead and reused by the four groups.
// Weights are copied into a per-lane shared-memory ring with cp.async (the whole ring requested before
// griddepcontrol.wait: weights never depend on the previous kernel).  With S > 1 each CTA writes its
// int32 partial tile to the workspace and the last CTA of a row tile to arrive (ticket counter, reset by
// that CTA) adds them and runs the epilogue.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

template <int WB, int NW>
struct DecShape {
  // ring depth in units: ~32 KB of weights in flight per 4-warp CTA (Little's law: ~40-60 KB per SM at
  // ~1 us of loaded HBM latency with ~2 CTAs per SM, leaving room for the next kernel's CTAs), at most 32
  static constexpr int kD0 = 8192 * 4 / (NW * WB * 256) * (NW >= 8 ? 2 : 1);
  static constexpr int kD = kD0 > 32 ? 32 : kD0 < 2 ? 2 : kD0;
  static constexpr int kShift = WB <= 2 ? 8 - WB : WB <= 4 ? 4 : 0;                // digits are u * 2^kShift
  static constexpr int kRingBytes = NW * kD * WB * 32 * 8;  // NW warps x D units x WB planes x 32 lanes x 8 B
  static constexpr int kRedBytes = (NW - 1) * 16 * 32 * 4;  // k-warp partial tiles
};

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
  // not volatile: a pure function of its operands, so the compiler may interleave one unit's MMAs with
  // the next unit's shared-memory loads and rebuild
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int WB>
__device__ __forceinline__ void dec_rebuild(const uint32_t* w, uint32_t (&o)[8]) {
  if constexpr (WB <= 2) rebuild_hi<WB>(w, o);
  else if constexpr (WB <= 4) rebuild_x16<WB>(w, o);
  else rebuild8<WB>(w, o);
}

#ifdef APT_DEC_TRACE
// per-warp globaltimer timeline (profiling builds only): [cta * 8 + warp][phase]; phases 0 entry,
// 1 prologue issued, 2 past griddepcontrol.wait, 3 first tokens landed, 4 first weights landed, 5 loop
// done, 6 ticket taken, 7 exit, 8 smid, 9 grid size, 10 partials summed (last CTA), 11 k-warps reduced
__device__ unsigned long long g_dec_trace[8192][12];
__device__ __forceinline__ unsigned long long dec_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define DTRACE(ph) do { if (lane == 0) { const unsigned c_ = (blockIdx.x + gridDim.x * blockIdx.z) * 8 + warp; \
  if (c_ < 8192) { g_dec_trace[c_][ph] = dec_gtimer(); if ((ph) == 0) { unsigned sm_; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_)); \
  g_dec_trace[c_][8] = sm_; g_dec_trace[c_][9] = gridDim.x * gridDim.z * 8; } } } } while (0)
#else
#define DTRACE(ph) do { } while (0)
#endif

template <int WB, int MT, int NW, bool TILED>
__global__ void __launch_bounds__(32 * NW, NW >= 8 ? 1 : 3) gemm_dec_kernel(DecArgs p) {
  using SH = DecShape<WB, NW>;
  constexpr int D = SH::kD;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ int s_last;
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  DTRACE(0);
  const int n_w = blockIdx.x * 32;  // first weight row of the CTA
  const int nb = p.k_words >> 3;    // 256-element K blocks
  const int S = gridDim.z;
  const int cb0 = (int)((int64_t)blockIdx.z * nb / S), cb1 = (int)((int64_t)(blockIdx.z + 1) * nb / S);
  const int b0 = cb0 + (cb1 - cb0) * warp / NW, b1 = cb0 + (cb1 - cb0) * (warp + 1) / NW;
  const int nblk = b1 - b0, U = nblk * 4;  // units = (block, group), block-major

  // ---- weight ring: [warp][slot][plane][lane] x 8 bytes; each lane reads back only its own copies
  const uint32_t ring = smem_u32(smem) + (uint32_t)(warp * D * WB * 32 * 8) + (uint32_t)lane * 8u;
  // per-plane source of unit (block b0, group 0); unit (b, q) adds b * blk_step + q * grp_step words
  const uint32_t* src0;
  int64_t blk_step, grp_step;
  if constexpr (TILED) {
    // tile-major: [plane][row tile][Kpad/256][2][128][4]; the CTA's 32 rows lie in one 128-row tile
    src0 = p.wp + ((int64_t)(n_w >> 7) * (p.k_words >> 3) + b0) * 1024 + (t >> 1) * 512 + ((n_w & 127) + g) * 4 + (t & 1) * 2;
    blk_step = 1024;
    grp_step = 32;
  } else {
    src0 = p.wp + (int64_t)min(n_w + g, p.e.N - 1) * p.k_words + b0 * 8 + 2 * t;
    blk_step = 8;
    grp_step = (int64_t)8 * p.k_words;
  }
  const int64_t pstride = p.w_pstride;
  auto issue = [&](int u) {
    if (u < U) {
      const int b = u >> 2, q = u & 3;
      const uint32_t* s = src0 + b * blk_step + q * grp_step;
      if constexpr (!TILED) {  // rows past N: clamp (their results are never stored)
        if (n_w + 8 * q + g >= p.e.N) s = p.wp + (int64_t)(p.e.N - 1) * p.k_words + (b0 + b) * 8 + 2 * t;
      }
      const uint32_t dst = ring + (uint32_t)((u % D) * WB * 256);
#pragma unroll
      for (int i = 0; i < WB; ++i) cp_async8(dst + (uint32_t)(i * 256), s + i * pstride);
    }
    cp_async_commit();  // empty groups keep the wait count uniform at the tail
  };
#pragma unroll 1
  for (int d = 0; d < D; ++d) issue(d);
  // weight-side epilogue operands (immutable, read before the wait like the planes): rows 8q + 2t + c
  int32_t rw[4][2];
  float wsc[4][2];
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int n = min(n_w + 8 * q + 2 * t + c, p.e.N - 1);
        rw[q][c] = __ldg(p.e.w_rowsum + n);
        wsc[q][c] = p.e.kind == 2 ? __ldg(p.e.w_scale + n) : 0.f;
      }
  }
  DTRACE(1);

  pdl_wait();  // the activation digit view / row sums / scales may come from the previous kernel
  DTRACE(2);
  // token-side epilogue operands
  int32_t ra[2];
  float as[2];
  if (warp == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = min(g + 8 * h, p.e.M - 1);
      ra[h] = __ldg(p.e.a_rowsum + m);
      as[h] = (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f;
    }
  }
  // ---- token fragments: rows g and g + 8 (clamped to M - 1; their output columns are never stored),
  // words 8b + 2t + c of the digit view, one block ahead
  const int64_t kp = (int64_t)p.k_words * 32;
  const uint4* tok0 = reinterpret_cast<const uint4*>(p.adig + (int64_t)min(g, p.e.M - 1) * kp) + 4 * t;
  const uint4* tok1 = reinterpret_cast<const uint4*>(p.adig + (int64_t)min(g + 8, p.e.M - 1) * kp) + 4 * t;
  auto load_tok = [&](int b, uint4 (&tk)[MT][4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // words 2t, 2t+1 of block b = 4 x 16 bytes
      tk[0][j] = __ldg(tok0 + b * 16 + j);
      if constexpr (MT > 1) tk[1][j] = __ldg(tok1 + b * 16 + j);
    }
  };

  int acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[q][j] = 0;
  // A fragments of the current block, assembled once per block as aligned quads {a0, a1, a2, a3} =
  // {row g reg 2s, row g+8 reg 2s, row g reg 2s+1, row g+8 reg 2s+1} of word 2t + c (no register moves
  // per MMA; rows >= 8 are zero for M <= 8)
  uint4 af[2][4];
  auto assemble = [&](const uint4 (&tk)[MT][4]) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint32_t* ag = reinterpret_cast<const uint32_t*>(&tk[0][2 * c]);
      const uint32_t* ah = reinterpret_cast<const uint32_t*>(&tk[MT - 1][2 * c]);
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4)
        af[c][s4] = make_uint4(ag[2 * s4], MT > 1 ? ah[2 * s4] : 0u, ag[2 * s4 + 1], MT > 1 ? ah[2 * s4 + 1] : 0u);
    }
  };
  if (nblk > 0) {
    uint4 tk[MT][4];
    load_tok(b0, tk);
    assemble(tk);
  }
#pragma unroll 1
  for (int bl = 0; bl < nblk; ++bl) {
    uint4 tn[MT][4];
    if (bl + 1 < nblk) load_tok(b0 + bl + 1, tn);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int u = bl * 4 + q;
      cp_async_wait<D - 1>();
      uint2 wv[WB];
      const uint32_t src = ring + (uint32_t)((u % D) * WB * 256);
#pragma unroll
      for (int i = 0; i < WB; ++i)
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(wv[i].x), "=r"(wv[i].y) : "r"(src + (uint32_t)(i * 256)) : "memory");
#ifdef APT_DEC_TRACE
      if (u == 0) DTRACE(4);
#endif
      issue(u + D);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t w[WB], o[8];
#pragma unroll
        for (int i = 0; i < WB; ++i) w[i] = c ? wv[i].y : wv[i].x;
        dec_rebuild<WB>(w, o);
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4)
          mma_u8(acc[q], af[c][s4].x, af[c][s4].y, af[c][s4].z, af[c][s4].w, o[2 * s4], o[2 * s4 + 1]);
      }
    }
    if (bl + 1 < nblk) assemble(tn);
  }
  cp_async_wait<0>();
  DTRACE(5);

  // ---- the NW warps of the CTA meet in shared memory (after the ring: [warp - 1][16][32])
  if constexpr (NW > 1) {
    int* red = reinterpret_cast<int*>(smem + SH::kRingBytes);
    if (warp > 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) red[((warp - 1) * 16 + j) * 32 + lane] = acc[j >> 2][j & 3];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        int v = acc[j >> 2][j & 3];
#pragma unroll
        for (int o = 0; o < NW - 1; ++o) v += red[(o * 16 + j) * 32 + lane];
        acc[j >> 2][j & 3] = v;
      }
    }
  }
  DTRACE(11);

  // ---- K split over CTAs: partials [tile][split][16][32] int32 in the workspace; the last CTA of the
  // tile to arrive (ticket) sums them and resets the ticket for the next call
  if (S > 1) {
    int* part = p.partials + (int64_t)blockIdx.x * S * 512;
    if (warp == 0) {
#pragma unroll
      for (int j = 0; j < 16; ++j) part[(int64_t)blockIdx.z * 512 + j * 32 + lane] = acc[j >> 2][j & 3];
    }
    // the CTA barrier orders warp 0's partial stores before thread 0's ticket; the ticket is an acq_rel
    // atomic at GPU scope (release: cumulative over those stores; acquire: the last CTA then sees every
    // other CTA's partials)
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(p.counters + blockIdx.x) : "memory");
      s_last = prev == (unsigned)(S - 1);
    }
    __syncthreads();
    DTRACE(6);
    if (!s_last) {
      DTRACE(7);
      return;
    }
    if (warp == 0) {
      // every split's partial (this CTA's own included, re-read from L2), 4 splits' loads in flight
      int tot[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) tot[j] = 0;
#pragma unroll 4
      for (int z = 0; z < S; ++z) {
#pragma unroll
        for (int j = 0; j < 16; ++j) tot[j] += __ldcg(part + (int64_t)z * 512 + j * 32 + lane);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j >> 2][j & 3] = tot[j];
    }
    DTRACE(10);
    if (threadIdx.x == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p.counters + blockIdx.x), "r"(0u) : "memory");
  }
  if (warp != 0) {
    DTRACE(7);
    return;
  }

  // ---- epilogue: acc[q] = U * 2^kShift for (token g | g+8) x (rows 8q + 2t, 8q + 2t + 1).  The output
  // kind is uniform: one branch outside the loops keeps the code (and its instruction-cache footprint,
  // paid once per CTA) small; both layouts through one address formula.
  const int64_t sm_ = p.e.layout == 0 ? p.e.ldo : 1, sn_ = p.e.layout == 0 ? 1 : p.e.ldo;
  const uint32_t kfix = (uint32_t)p.e.kpad * (uint32_t)p.e.h_a * (uint32_t)p.e.h_w;
  if (p.e.kind == 2) {
    unsigned short* out = reinterpret_cast<unsigned short*>(p.e.out);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int q = j >> 2, h = (j >> 1) & 1, c = j & 1;
      const int m = g + 8 * h, n = n_w + 8 * q + 2 * t + c;
      const uint32_t y = (((uint32_t)acc[q][2 * h + c]) >> SH::kShift) - (uint32_t)p.e.h_w * (uint32_t)ra[h] -
                         (uint32_t)p.e.h_a * (uint32_t)rw[q][c] - kfix;
      const float v = ((float)(int32_t)y * wsc[q][c]) * as[h];
      unsigned short hv;
      asm("cvt.rn.f16.f32 %0, %1;" : "=h"(hv) : "f"(v));
      if (m < p.e.M && n < p.e.N) out[m * sm_ + n * sn_] = hv;
    }
  } else {
    int32_t* out = reinterpret_cast<int32_t*>(p.e.out);
    const bool bip = p.e.kind == 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int q = j >> 2, h = (j >> 1) & 1, c = j & 1;
      const int m = g + 8 * h, n = n_w + 8 * q + 2 * t + c;
      const uint32_t y = (((uint32_t)acc[q][2 * h + c]) >> SH::kShift) - (uint32_t)p.e.h_w * (uint32_t)ra[h] -
                         (uint32_t)p.e.h_a * (uint32_t)rw[q][c] - kfix;
      const uint32_t yb = 4u * y + 2u * (uint32_t)ra[h] + 2u * (uint32_t)rw[q][c] + (uint32_t)p.e.K;  // Y' (I2)
      if (m < p.e.M && n < p.e.N) out[m * sm_ + n * sn_] = (int32_t)(bip ? yb : y);
    }
  }
  DTRACE(7);
}

int dec_blocks_per_cta(int k_words, int split) { return ((k_words >> 3) + split - 1) / split; }

template <int WB, int MT, int NW, bool TILED>
static cudaError_t launch_dec4(const DecArgs& p, int split, cudaStream_t stream) {
  using SH = DecShape<WB, NW>;
  constexpr int kSmem = SH::kRingBytes + SH::kRedBytes;
  cudaError_t err = set_smem_once<gemm_dec_kernel<WB, MT, NW, TILED>>(kSmem);
  if (err != cudaSuccess) return err;
  const dim3 grid((p.e.N + 31) / 32, 1, split);
  return launch_pdl(gemm_dec_kernel<WB, MT, NW, TILED>, grid, dim3(32 * NW), kSmem, stream, dim3(1, 1, 1), p);
}

template <int WB, int MT>
static cudaError_t launch_dec2(const DecArgs& p, int warps, int split, cudaStream_t stream) {
  if (warps == 8) return p.w_tiled ? launch_dec4<WB, MT, 8, true>(p, split, stream) : launch_dec4<WB, MT, 8, false>(p, split, stream);
  return p.w_tiled ? launch_dec4<WB, MT, 4, true>(p, split, stream) : launch_dec4<WB, MT, 4, false>(p, split, stream);
}

template <int WB>
static cudaError_t launch_dec1(const DecArgs& p, int warps, int split, cudaStream_t stream) {
  return p.e.M > 8 ? launch_dec2<WB, 2>(p, warps, split, stream) : launch_dec2<WB, 1>(p, warps, split, stream);
}

cudaError_t launch_gemm_dec(const DecArgs& p, int wbits, int warps, int split, cudaStream_t stream) {
  switch (wbits) {
    case 1: return launch_dec1<1>(p, warps, split, stream);
    case 2: return launch_dec1<2>(p, warps, split, stream);
    case 3: return launch_dec1<3>(p, warps, split, stream);
    case 4: return launch_dec1<4>(p, warps, split, stream);
    case 5: return launch_dec1<5>(p, warps, split, stream);
    case 6: return launch_dec1<6>(p, warps, split, stream);
    case 7: return launch_dec1<7>(p, warps, split, stream);
    default: return launch_dec1<8>(p, warps, split, stream);
  }
}

size_t dec_workspace_bytes(int N, int split) {
  if (split <= 1) return 0;
  // partials [tile][split][16][32] int32 (the tickets live in the workspace's fixed ticket area)
  return (size_t)((N + 31) / 32) * (size_t)split * 512u * 4u;
}

}  // namespace apt

#ifdef APT_DEC_TRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_dec_trace(unsigned long long* host, int n, int reset) {
  if (reset) {
    static unsigned long long zero[8192 * 12];
    return (int)cudaMemcpyToSymbol(apt::g_dec_trace, zero, sizeof(zero));
  }
  return (int)cudaMemcpyFromSymbol(host, apt::g_dec_trace, sizeof(unsigned long long) * (n < 8192 * 12 ? n : 8192 * 12));
}
#endif
