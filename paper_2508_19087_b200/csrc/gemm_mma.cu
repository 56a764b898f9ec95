// gemm_mma.cu — APT W_p x A_q GEMM for small token counts (decode, M <= 64): register rebuild of
// the weight planes into u8 digit fragments + legacy mma.sync.m16n8k32.u8.u8.s32, K split across the
// warps of a CTA and reduced through shared memory.
//
// Mapping to the paper:
//   * recovery-oriented scheduling (§4.2 (1)): every plane of a B_M x B_N output block is
//     consumed in one CTA and nothing per-plane reaches global memory;
//   * K partitioned into B_K steps (§4.2 (2)) and "weight-bit fragment reuse" (§4.2 (4),
//     P:276): the weight planes of a 16-row fragment are rebuilt once per K step and reused for every
//     8-token MMA column tile;
//   * the shift-add of P:228 is folded into the operand rebuild (digit = sum_i 2^i u_i), so each
//     K=32 step is ONE u8 MMA for any p, q <= 8 instead of p*q 1-bit MMAs (R1);
//   * the remaining rank-1 terms and the fp16 scale are applied in the epilogue (common.cuh).
//
// Decode is a stream over the packed weights, so the kernel is a flat latency chain:
//   CTA = W warps (W = split_k <= 8) x 16 weight rows (one MMA M tile) x BN = 8*NT tokens.  Warp w owns
//   a contiguous 1/W of K.  Every lane loads its own 32-byte sector quarter of the plane words of rows
//   g and g+8 (each packed weight byte is loaded exactly once, straight into registers, one
//   256-element iteration ahead) and the activation digits (kernel-order u8, L2 resident) for the
//   same K; it rebuilds the weight fragments with rebuild8() and issues the MMAs.  The W partial
//   16 x BN tiles are summed through shared memory and stored by the epilogue, whose operands (row
//   sums, scales) were requested at kernel entry.  No cluster, no global atomics, one __syncthreads.
//
// K order inside the MMA: an iteration covers 8 plane words (256 K elements) of a row.  Lane (g, t)
// owns words 2t (group 0) and 2t+1 (group 1); the 8 digit registers of rebuild8() for a word fill the
// 4 K=32 steps of its group (reg 2s -> a0/a1/b0, reg 2s+1 -> a2/a3/b1).  The activation digit view is
// written by the pack kernel (or the expand pre-pass) with the same rebuild8() order, so both
// operands agree on K.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace apt {

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream_v2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

#ifdef APT_MMA_TRACE
// globaltimer per CTA: [cta][phase] (profiling builds only)
__device__ unsigned long long g_mma_trace[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define MTRACE(ph) do { if (threadIdx.x == 0) { const int c_ = blockIdx.x + gridDim.x * blockIdx.y; if (c_ < 4096) g_mma_trace[c_][ph] = gtimer(); } } while (0)
#else
#define MTRACE(ph) do { } while (0)
#endif

template <int WB, int NT>
struct DecIter {
  uint2 w0[WB], w1[WB];  // plane words 2t, 2t+1 of rows g and g+8
  uint4 b[NT][4];        // activation digits of words 2t, 2t+1 (32 B each) for token nt*8+g
};

template <int WB, int NT>
__device__ __forceinline__ void dec_load(DecIter<WB, NT>& d, const uint32_t* w0p, const uint32_t* w1p, bool ok0,
                                         bool ok1, int64_t pstride, const uint8_t* const (&bp)[NT],
                                         const bool (&bok)[NT], int word0) {
#pragma unroll
  for (int i = 0; i < WB; ++i) {
    d.w0[i] = ok0 ? ldg_stream_v2(w0p + (int64_t)i * pstride + word0) : make_uint2(0, 0);
    d.w1[i] = ok1 ? ldg_stream_v2(w1p + (int64_t)i * pstride + word0) : make_uint2(0, 0);
  }
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      d.b[nt][q] = bok[nt] ? ldg_nc_v4(bp[nt] + (size_t)word0 * 32 + 16 * q) : make_uint4(0, 0, 0, 0);
  }
}

template <int WB, int NT>
__global__ void __launch_bounds__(256) gemm_mma_kernel(MmaArgs p) {
  constexpr int BN = NT * 8;
  __shared__ int32_t red[8][16][BN];

  MTRACE(0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int N = p.e.N, M = p.e.M;
  const int n0 = blockIdx.x * 16;
  const int tok0 = blockIdx.y * BN;
  const int n_it = p.k_words >> 3;
  const int it_b = (warp * n_it) / nwarps, it_e = ((warp + 1) * n_it) / nwarps;
  const int kpad_bytes = p.k_words * 32;

  // epilogue operands, requested first (consumed at the very end)
  const int e_row = tid & 15, e_tok = tid >> 4;  // thread -> (row, token) of the 16 x BN tile
  const bool e_act = e_tok < BN && n0 + e_row < N && tok0 + e_tok < M;
  int32_t e_rw = 0, e_ra = 0;
  float e_ws = 0.f, e_as = 1.f;
  if (e_act) {
    e_rw = __ldg(p.e.w_rowsum + n0 + e_row);
    e_ra = __ldg(p.e.a_rowsum + tok0 + e_tok);
    if (p.e.kind == 2) {
      e_ws = __ldg(p.e.w_scale + n0 + e_row);
      if (p.e.a_scale) e_as = __ldg(p.e.a_scale + tok0 + e_tok);
    }
  }

  const bool ok0 = n0 + g < N, ok1 = n0 + g + 8 < N;
  const uint32_t* w0p = p.wp + (int64_t)(ok0 ? n0 + g : 0) * p.k_words + 2 * t;
  const uint32_t* w1p = p.wp + (int64_t)(ok1 ? n0 + g + 8 : 0) * p.k_words + 2 * t;
  const uint8_t* bp[NT];
  bool bok[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int tok = tok0 + nt * 8 + g;
    bok[nt] = tok < M;
    bp[nt] = p.adig + (size_t)(bok[nt] ? tok : 0) * kpad_bytes + 2 * t * 32;
  }

  int acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;

  DecIter<WB, NT> cur, nxt;
  if (it_b < it_e) dec_load<WB, NT>(cur, w0p, w1p, ok0, ok1, p.w_pstride, bp, bok, it_b * 8);
  MTRACE(1);
  for (int it = it_b; it < it_e; ++it) {
    if (it + 1 < it_e) dec_load<WB, NT>(nxt, w0p, w1p, ok0, ok1, p.w_pstride, bp, bok, (it + 1) * 8);
#pragma unroll
    for (int gr = 0; gr < 2; ++gr) {
      uint32_t wa[WB], wb[WB], ra[8], rb[8];
#pragma unroll
      for (int i = 0; i < WB; ++i) {
        wa[i] = gr ? cur.w0[i].y : cur.w0[i].x;
        wb[i] = gr ? cur.w1[i].y : cur.w1[i].x;
      }
      rebuild8<WB>(wa, ra);
      rebuild8<WB>(wb, rb);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          // digits of word 2t+gr, registers 2s and 2s+1: uint4 index gr*2 + s/2, components (s%2)*2, +1
          const uint4 q = cur.b[nt][gr * 2 + (s >> 1)];
          const uint32_t b0 = (s & 1) ? q.z : q.x;
          const uint32_t b1 = (s & 1) ? q.w : q.y;
          mma_u8(acc[nt], ra[2 * s], rb[2 * s], ra[2 * s + 1], rb[2 * s + 1], b0, b1);
        }
      }
    }
    if (it + 1 < it_e) cur = nxt;
  }
  MTRACE(2);

  // ---- reduction of the per-warp K partials through shared memory
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int tk = nt * 8 + 2 * t;
    red[warp][g][tk] = acc[nt][0];
    red[warp][g][tk + 1] = acc[nt][1];
    red[warp][g + 8][tk] = acc[nt][2];
    red[warp][g + 8][tk + 1] = acc[nt][3];
  }
  __syncthreads();
  MTRACE(3);
  if (e_act) {
    uint32_t U = 0;
    for (int w = 0; w < nwarps; ++w) U += (uint32_t)red[w][e_row][e_tok];
    epilogue_store_v(p.e, tok0 + e_tok, n0 + e_row, U, e_ra, e_rw, e_ws, e_as);
  }
  MTRACE(4);
}

template <int WB, int NT>
static cudaError_t launch_one(const MmaArgs& p, int warps, cudaStream_t stream) {
  dim3 grid((p.e.N + 15) / 16, (p.e.M + NT * 8 - 1) / (NT * 8));
  gemm_mma_kernel<WB, NT><<<grid, 32 * warps, 0, stream>>>(p);
  return cudaGetLastError();
}

template <int WB>
static cudaError_t launch_wb(const MmaArgs& p, int nt, int warps, cudaStream_t stream) {
  switch (nt) {
    case 1: return launch_one<WB, 1>(p, warps, stream);
    case 2: return launch_one<WB, 2>(p, warps, stream);
    case 4: return launch_one<WB, 4>(p, warps, stream);
    default: return launch_one<WB, 8>(p, warps, stream);
  }
}

cudaError_t launch_gemm_mma(const MmaArgs& p, int wbits, int bn, int warps, cudaStream_t stream) {
  const int nt = bn / 8;
  // the epilogue maps one thread per (row, token) of the 16 x BN tile
  if (warps * 32 < 16 * bn) warps = (16 * bn) / 32;
  switch (wbits) {
    case 1: return launch_wb<1>(p, nt, warps, stream);
    case 2: return launch_wb<2>(p, nt, warps, stream);
    case 3: return launch_wb<3>(p, nt, warps, stream);
    case 4: return launch_wb<4>(p, nt, warps, stream);
    case 5: return launch_wb<5>(p, nt, warps, stream);
    case 6: return launch_wb<6>(p, nt, warps, stream);
    case 7: return launch_wb<7>(p, nt, warps, stream);
    default: return launch_wb<8>(p, nt, warps, stream);
  }
}

}  // namespace apt

#ifdef APT_MMA_TRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_mma_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, apt::g_mma_trace, sizeof(unsigned long long) * (n < 4096 * 8 ? n : 4096 * 8));
}
#endif
