// gemm_mma.cu — APT W_p x A_q GEMM for small token counts (decode, M <= 64): TMA-streamed weight
// bit-planes, register rebuild into u8 digit fragments + legacy mma.sync.m16n8k32.u8.u8.s32, K split
// across the warps of a CTA and reduced through shared memory.
//
// Mapping to the paper:
//   * recovery-oriented scheduling (§4.2 (1)): every plane of a B_M x B_N output block is
//     consumed in one CTA and nothing per-plane reaches global memory;
//   * the unified matrix moves with single commands (§4.1 Step 3): one 3-D TMA box carries all
//     wbits planes of a 16-row x 256-element weight slab;
//   * K partitioned into B_K steps with multi-buffered staging (§4.2 (2)/(3)) and
//     "weight-bit fragment reuse" (§4.2 (4)): a 16-row weight fragment is rebuilt once per K step
//     and reused for every 8-token MMA column tile; the activation planes of the CTA's tokens are staged
//     once in shared memory;
//   * the shift-add of P:228 is folded into the operand rebuild (digit = sum_i 2^i u_i), so each
//     K=32 step is ONE u8 MMA for any p, q <= 8 instead of p*q 1-bit MMAs (R1);
//   * the remaining rank-1 terms and the fp16 scale are applied in the epilogue (common.cuh).
//
// Decode streams the packed weights once and is bound by bytes in flight, so every warp owns a
// private `depth`-slot TMA ring: CTA = 8 warps = 2 row tiles (16 weight rows, the MMA M side) x 4 K
// quarters, BN = 8*NT tokens.  Lane 0 of each warp keeps `depth` 256-element slabs of its (row tile,
// K quarter) in flight (mbarrier complete_tx), refilling a slot as soon as the warp has read it.
// The four K-quarter partials are summed through shared memory and stored by the epilogue, whose
// operands were requested at entry.
//
// K order inside the MMA: an iteration covers 8 plane words (256 K elements) of a row.  Lane (g, t)
// owns words 2t (group 0) and 2t+1 (group 1); the 8 digit registers of rebuild8() for a word fill the
// 4 K=32 steps of its group (reg 2s -> a0/a1/b0, reg 2s+1 -> a2/a3/b1).  Tokens go through the same
// rebuild8() of the same word, so both operands agree on K.
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

constexpr int kDecRows = 32;      // weight rows per CTA (2 MMA M tiles)
constexpr int kDecKq = 4;         // K quarters per CTA
constexpr int kDecThreads = 256;  // 8 warps
constexpr int kDecWarps = 8;
constexpr int kDecMaxSmem = 220 * 1024;

// token-plane row pitch in u32 words: >= k_words and == 8 (mod 32), so the 8 token rows a warp reads
// with one 64-bit load land in distinct bank groups (2 wavefronts for 256 B, the minimum)
__host__ __device__ inline int dec_stride(int k_words) { return k_words + ((8 - (k_words & 31)) & 31); }

struct DecSmem {
  int ring_off, tok_off, red_off, ep_off, bar_off, total;
};

// rings [8 warps][depth][wbits][16 rows][8 words] | token planes [abits][BN][stride] |
// partials [4][32][BN] | epilogue operands | mbarriers [8][depth]
__host__ __device__ inline DecSmem dec_smem_layout(int wbits, int abits, int bn, int k_words, int depth) {
  DecSmem L;
  L.ring_off = 0;
  L.tok_off = L.ring_off + kDecWarps * depth * wbits * 512;
  L.red_off = L.tok_off + abits * bn * dec_stride(k_words) * 4;
  L.ep_off = L.red_off + kDecKq * kDecRows * bn * 4;
  L.bar_off = (L.ep_off + (2 * kDecRows + 2 * bn) * 4 + 7) & ~7;
  L.total = L.bar_off + kDecWarps * depth * 8;
  return L;
}

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
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
__global__ void __launch_bounds__(kDecThreads) gemm_mma_kernel(const __grid_constant__ CUtensorMap tm_w, MmaArgs p) {
  constexpr int BN = NT * 8;
  constexpr uint32_t kSlab = WB * 512;  // bytes of one 16-row x 256-element slab, all planes
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int kw = p.k_words;
  const int D = p.depth;
  const DecSmem L = dec_smem_layout(WB, p.abits, BN, kw, D);
  const int stride = dec_stride(kw);
  uint32_t* sT = reinterpret_cast<uint32_t*>(smem_raw + L.tok_off);
  int32_t* red = reinterpret_cast<int32_t*>(smem_raw + L.red_off);
  int32_t* ep_rw = reinterpret_cast<int32_t*>(smem_raw + L.ep_off);
  float* ep_ws = reinterpret_cast<float*>(ep_rw + kDecRows);
  int32_t* ep_ra = reinterpret_cast<int32_t*>(ep_ws + kDecRows);
  float* ep_as = reinterpret_cast<float*>(ep_ra + BN);

  MTRACE(0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int rt = warp & 1, kq = warp >> 1;  // row tile, K quarter
  const int N = p.e.N, M = p.e.M;
  const int n0 = blockIdx.x * kDecRows;
  const int tok0 = blockIdx.y * BN;
  const int n_it = kw >> 3;
  const int it_b = (kq * n_it) / kDecKq, it_e = ((kq + 1) * n_it) / kDecKq;
  const int n_my = it_e - it_b;
  const uint32_t ring = smem_u32(smem_raw + L.ring_off) + (uint32_t)(warp * D) * kSlab;
  const uint32_t bars = smem_u32(smem_raw + L.bar_off) + (uint32_t)(warp * D) * 8u;

  pdl_launch_dependents();
  // 1. this warp's weight slabs in flight (TMA, one box = all planes of 16 rows x 256 elements)
  if (lane == 0) {
    for (int d = 0; d < D; ++d) mbar_init(bars + 8 * d, 1);
    fence_proxy_async();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_w) : "memory");
    for (int j = 0; j < D && j < n_my; ++j) {
      mbar_expect_tx(bars + 8 * j, kSlab);
      tma_load_3d(ring + j * kSlab, &tm_w, bars + 8 * j, (it_b + j) * 8, n0 + rt * 16, 0);
    }
  }
  pdl_wait();  // activations / outputs may belong to the previous kernel
  // 2. the CTA's token planes -> shared memory (cp.async, 16 B chunks), rows beyond M zero-filled
  {
    const int chunks_per_row = kw >> 2;
    const int total = p.abits * BN * chunks_per_row;
    const uint32_t s_base = smem_u32(sT);
    for (int c = tid; c < total; c += kDecThreads) {
      const int row = c / chunks_per_row, ch = c - row * chunks_per_row;  // row = plane * BN + token
      const int plane = row / BN, tk = row - plane * BN;
      const int tok = tok0 + tk;
      const uint32_t* src = p.ap + (int64_t)plane * p.a_pstride + (int64_t)(tok < M ? tok : 0) * kw + 4 * ch;
      cp_async16(s_base + (uint32_t)((row * stride + 4 * ch) * 4), src, tok < M ? 16u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // 3. epilogue operands
  if (tid < kDecRows) {
    const int n = min(n0 + tid, N - 1);
    ep_rw[tid] = __ldg(p.e.w_rowsum + n);
    ep_ws[tid] = p.e.kind == 2 ? __ldg(p.e.w_scale + n) : 0.f;
  } else if (tid - kDecRows < BN) {
    const int m = min(tok0 + tid - kDecRows, M - 1);
    ep_ra[tid - kDecRows] = __ldg(p.e.a_rowsum + m);
    ep_as[tid - kDecRows] = (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  MTRACE(1);

  int acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;

  for (int j = 0; j < n_my; ++j) {
    const int it = it_b + j;
    const int slot = j % D;
    mbar_wait(bars + 8 * slot, (uint32_t)((j / D) & 1));
    // weight words 2t, 2t+1 of rows g and g+8 of every plane (conflict-free 64-bit reads)
    const uint8_t* sl = smem_raw + L.ring_off + (size_t)(warp * D + slot) * kSlab;
    uint2 w0[WB], w1[WB];
#pragma unroll
    for (int i = 0; i < WB; ++i) {
      w0[i] = *reinterpret_cast<const uint2*>(sl + (i * 16 + g) * 32 + 8 * t);
      w1[i] = *reinterpret_cast<const uint2*>(sl + (i * 16 + g + 8) * 32 + 8 * t);
    }
    __syncwarp();
    if (lane == 0 && j + D < n_my) {  // refill the slot this warp just drained
      fence_proxy_async();
      mbar_expect_tx(bars + 8 * slot, kSlab);
      tma_load_3d(ring + slot * kSlab, &tm_w, bars + 8 * slot, (it + D) * 8, n0 + rt * 16, 0);
    }
    // token fragments: words 2t, 2t+1 of token nt*8+g, every plane, rebuilt to digits
    uint32_t tb[NT][2][8];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      uint32_t lo[8], hi[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < p.abits) {
          const uint2 v = *reinterpret_cast<const uint2*>(sT + (i * BN + nt * 8 + g) * stride + it * 8 + 2 * t);
          lo[i] = v.x;
          hi[i] = v.y;
        } else {
          lo[i] = hi[i] = 0u;
        }
      }
      rebuild8_rt(lo, p.abits, tb[nt][0]);
      rebuild8_rt(hi, p.abits, tb[nt][1]);
    }
#pragma unroll
    for (int gr = 0; gr < 2; ++gr) {
      uint32_t wa[WB], wb[WB], ra[8], rb[8];
#pragma unroll
      for (int i = 0; i < WB; ++i) {
        wa[i] = gr ? w0[i].y : w0[i].x;
        wb[i] = gr ? w1[i].y : w1[i].x;
      }
      rebuild8<WB>(wa, ra);
      rebuild8<WB>(wb, rb);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          mma_u8(acc[nt], ra[2 * s], rb[2 * s], ra[2 * s + 1], rb[2 * s + 1], tb[nt][gr][2 * s],
                 tb[nt][gr][2 * s + 1]);
      }
    }
  }
  MTRACE(2);

  // ---- the four K-quarter partials meet in shared memory
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int tk = nt * 8 + 2 * t;
    const int lr = rt * 16 + g;
    red[(kq * kDecRows + lr) * BN + tk] = acc[nt][0];
    red[(kq * kDecRows + lr) * BN + tk + 1] = acc[nt][1];
    red[(kq * kDecRows + lr + 8) * BN + tk] = acc[nt][2];
    red[(kq * kDecRows + lr + 8) * BN + tk + 1] = acc[nt][3];
  }
  __syncthreads();
  MTRACE(3);
  for (int idx = tid; idx < kDecRows * BN; idx += kDecThreads) {
    int lr, tk;
    if (p.e.layout == 0) { lr = idx % kDecRows; tk = idx / kDecRows; }  // consecutive rows n -> coalesced
    else { tk = idx % BN; lr = idx / BN; }                            // consecutive tokens m -> coalesced
    const int n = n0 + lr, m = tok0 + tk;
    if (n < N && m < M) {
      uint32_t U = 0;
#pragma unroll
      for (int q = 0; q < kDecKq; ++q) U += (uint32_t)red[(q * kDecRows + lr) * BN + tk];
      epilogue_store_v(p.e, m, n, U, ep_ra[tk], ep_rw[lr], ep_ws[lr], ep_as[tk]);
    }
  }
  MTRACE(4);
}

// deepest per-warp ring (2..8 slabs) that fits next to the token planes; 0 if even 2 do not fit
int mma_depth(int wbits, int abits, int bn, int k_words) {
  for (int d = 8; d >= 2; --d)
    if (dec_smem_layout(wbits, abits, bn, k_words, d).total <= kDecMaxSmem) return d;
  return 0;
}

template <int WB, int NT>
static cudaError_t launch_one(const CUtensorMap& tw, const MmaArgs& p, cudaStream_t stream) {
  const int smem = dec_smem_layout(WB, p.abits, NT * 8, p.k_words, p.depth).total;
  auto kern = gemm_mma_kernel<WB, NT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (err != cudaSuccess) return err;
  dim3 grid((p.e.N + kDecRows - 1) / kDecRows, (p.e.M + NT * 8 - 1) / (NT * 8));
  return launch_pdl(kern, grid, dim3(kDecThreads), smem, stream, dim3(1, 1, 1), tw, p);
}

template <int WB>
static cudaError_t launch_wb(const CUtensorMap& tw, const MmaArgs& p, int nt, cudaStream_t stream) {
  return nt == 1 ? launch_one<WB, 1>(tw, p, stream) : launch_one<WB, 2>(tw, p, stream);
}

cudaError_t launch_gemm_mma(const MmaArgs& p_in, int wbits, int bn, cudaStream_t stream) {
  MmaArgs p = p_in;
  p.depth = mma_depth(wbits, p.abits, bn, p.k_words);
  if (p.depth < 2) return cudaErrorInvalidConfiguration;
  CUtensorMap tw;
  if (!make_plane_map(&tw, p.wp, p.k_words, p.e.N, wbits, 8, 16)) return cudaErrorInvalidValue;
  const int nt = bn / 8;
  switch (wbits) {
    case 1: return launch_wb<1>(tw, p, nt, stream);
    case 2: return launch_wb<2>(tw, p, nt, stream);
    case 3: return launch_wb<3>(tw, p, nt, stream);
    case 4: return launch_wb<4>(tw, p, nt, stream);
    case 5: return launch_wb<5>(tw, p, nt, stream);
    case 6: return launch_wb<6>(tw, p, nt, stream);
    case 7: return launch_wb<7>(tw, p, nt, stream);
    default: return launch_wb<8>(tw, p, nt, stream);
  }
}

}  // namespace apt

#ifdef APT_MMA_TRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_mma_trace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, apt::g_mma_trace, sizeof(unsigned long long) * (n < 4096 * 8 ? n : 4096 * 8));
}
#endif
