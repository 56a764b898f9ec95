// gemm_mma.cu — APT W_p x A_q GEMM for small token counts (decode, M <= 64): register rebuild of
// the weight planes into u8 digit fragments + legacy mma.sync.m16n8k32.u8.u8.s32, split-K across a
// thread-block cluster and reduced through distributed shared memory.
//
// Mapping to the paper:
//   * recovery-oriented scheduling (§4.2 (1)): every plane of a B_M x B_N output block is
//     consumed in one CTA and nothing per-plane reaches global memory;
//   * K partitioned into B_K steps (§4.2 (2)) and "weight-bit fragment reuse" (§4.2 (4),
//     P:276): the weight planes of a 16-row fragment are rebuilt once per K step and reused for every
//     8-token MMA column tile;
//   * the shift-add of P:228 is folded into the operand rebuild (digit = sum_i 2^i u_i), so each
//     K=32 step is ONE u8 MMA for any p, q <= 8 instead of p*q 1-bit MMAs;
//   * the remaining rank-1 terms and the fp16 scale are applied in the epilogue (common.cuh).
//
// CTA = 4 warps = 64 weight rows (16 per warp, the MMA M side) x BN = 8*NT tokens (MMA N side).
// grid = (ceil(N/64), ceil(M/BN), split_k); cluster = (1, 1, split_k).  Each CTA of a cluster sums a
// contiguous K range; rank 0 reduces the partial tiles over DSMEM and runs the epilogue.
//
// K order inside the MMA: an iteration covers 8 plane words (256 K elements) of a row.  Lane (g, t)
// owns words kw0 + 2t (group 0) and kw0 + 2t + 1 (group 1) of rows g and g+8; the 8 digit registers of
// rebuild8() for that word fill the 4 K=32 steps of its group (reg 2s -> a0/a1/b0, reg 2s+1 ->
// a2/a3/b1).  Tokens use the identical mapping (pre-rebuilt into shared memory), so the sum over K is
// unchanged while every weight byte is loaded exactly once, 32 bytes per quad (one sector).
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace apt {


constexpr int kKch = 32;   // plane words (1024 K elements) of tokens staged per chunk

__device__ __forceinline__ void mma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// shared-memory index of token digit pair {reg 2s, reg 2s+1} for (iteration it, group gr, step s,
// token n, lane-in-quad t)
__device__ __forceinline__ int sb_index(int it, int gr, int s, int n, int t, int bn) {
  return (((it * 2 + gr) * 4 + s) * bn + n) * 4 + t;
}

template <int WB, int NT>
__global__ void __launch_bounds__(128) gemm_mma_kernel(MmaArgs p) {
  constexpr int BN = NT * 8;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint2* sB = reinterpret_cast<uint2*>(smem_raw);                          // token digits, kKch words
  int32_t* rbuf = reinterpret_cast<int32_t*>(smem_raw + (size_t)kKch * 32 * BN);  // [S][slots][64] partials

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int N = p.e.N, M = p.e.M;
  const int S = gridDim.z;
  const int slots = (BN + S - 1) / S;                      // tokens owned per rank in the reduction
  const int row0 = blockIdx.x * 64 + warp * 16 + g;        // rows row0 and row0 + 8
  const int tok0 = blockIdx.y * BN;
  const uint32_t rank = (S > 1) ? cluster_ctarank() : 0u;
  // every CTA of the cluster must have started before anyone stores into its shared memory:
  // arrive now, wait just before the reduction pushes (overlaps with the whole K loop)
  if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  const int kw_begin = (int)rank * p.kw_per_split;
  const int kw_end = min(p.k_words, kw_begin + p.kw_per_split);
  const int n_it = kw_end > kw_begin ? (kw_end - kw_begin) >> 3 : 0;

  const bool ok0 = row0 < N, ok1 = row0 + 8 < N;
  const uint32_t* w0 = p.wp + (int64_t)(ok0 ? row0 : 0) * p.k_words + 2 * t + kw_begin;
  const uint32_t* w1 = p.wp + (int64_t)(ok1 ? row0 + 8 : 0) * p.k_words + 2 * t + kw_begin;

  int acc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;

  // first iteration's weight words are requested before anything else (HBM latency is the bound)
  uint2 cur0[WB], cur1[WB];
#pragma unroll
  for (int i = 0; i < WB; ++i) {
    cur0[i] = (n_it > 0 && ok0) ? __ldg(reinterpret_cast<const uint2*>(w0 + (int64_t)i * p.w_pstride)) : make_uint2(0, 0);
    cur1[i] = (n_it > 0 && ok1) ? __ldg(reinterpret_cast<const uint2*>(w1 + (int64_t)i * p.w_pstride)) : make_uint2(0, 0);
  }
  constexpr int kItPerChunk = kKch / 8;
  for (int gi = 0; gi < n_it; ++gi) {
    const int it = gi % kItPerChunk;
    if (it == 0) {
      // ---- token rebuild: planes -> u8 digits in the MMA K order, once per CTA chunk
      const int chunk = kw_begin + gi * 8;
      const int nwc = min(kKch, kw_end - chunk);
      __syncthreads();
      for (int idx = threadIdx.x; idx < BN * nwc; idx += blockDim.x) {
        const int n = idx / nwc, o = idx - n * nwc;
        const int tok = tok0 + n;
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
          w[i] = (i < p.abits && tok < M)
                     ? __ldg(p.ap + (int64_t)i * p.a_pstride + (int64_t)tok * p.k_words + chunk + o) : 0u;
        uint32_t d[8];
        rebuild8_rt(w, p.abits, d);
        const int iq = o >> 3, r = o & 7, tt = r >> 1, gr = r & 1;
#pragma unroll
        for (int s = 0; s < 4; ++s) sB[sb_index(iq, gr, s, n, tt, BN)] = make_uint2(d[2 * s], d[2 * s + 1]);
      }
      __syncthreads();
    }
    // ---- prefetch the next 8 plane words of both rows, then rebuild + MMA on the current ones
    uint2 nxt0[WB], nxt1[WB];
    const bool more = gi + 1 < n_it;
#pragma unroll
    for (int i = 0; i < WB; ++i) {
      const int64_t off = (int64_t)i * p.w_pstride + (gi + 1) * 8;
      nxt0[i] = (more && ok0) ? __ldg(reinterpret_cast<const uint2*>(w0 + off)) : make_uint2(0, 0);
      nxt1[i] = (more && ok1) ? __ldg(reinterpret_cast<const uint2*>(w1 + off)) : make_uint2(0, 0);
    }
#pragma unroll
    for (int gr = 0; gr < 2; ++gr) {
      uint32_t wa[WB], wb[WB], ra[8], rb[8];
#pragma unroll
      for (int i = 0; i < WB; ++i) {
        wa[i] = gr ? cur0[i].y : cur0[i].x;
        wb[i] = gr ? cur1[i].y : cur1[i].x;
      }
      rebuild8<WB>(wa, ra);
      rebuild8<WB>(wb, rb);
#pragma unroll
      for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint2 b = sB[sb_index(it, gr, s, j * 8 + g, t, BN)];
          mma_u8(acc[j], ra[2 * s], rb[2 * s], ra[2 * s + 1], rb[2 * s + 1], b.x, b.y);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < WB; ++i) { cur0[i] = nxt0[i]; cur1[i] = nxt1[i]; }
  }

  // ---- split-K reduction: every partial is pushed (DSMEM store) to the rank that owns its token
  //      (owner = token % S), one cluster barrier, then each rank sums its slice and stores it.
  const int lrow = warp * 16 + g;
  const uint32_t rb_local = smem_u32(rbuf);
  if (S > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < NT; ++j) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int tk = j * 8 + 2 * t + (h & 1);
      const int lr = lrow + (h >> 1) * 8;
      const int owner = tk % S, slot = tk / S;
      const uint32_t off = (uint32_t)((((int)rank * slots + slot) * 64 + lr) * 4);
      if (S > 1) {
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(rb_local + off), "r"(owner));
        asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(acc[j][h]) : "memory");
      } else {
        rbuf[off / 4] = acc[j][h];
      }
    }
  }
  if (S > 1) cluster_sync_all(); else __syncthreads();
  const int mine = (BN - (int)rank + S - 1) / S;  // tokens tk = rank + S*slot < BN
  for (int idx = threadIdx.x; idx < mine * 64; idx += blockDim.x) {
    int slot, lr;
    if (p.e.layout == 0) { slot = idx >> 6; lr = idx & 63; }   // consecutive rows n -> coalesced
    else { slot = idx % mine; lr = idx / mine; }
    const int tk = (int)rank + S * slot;
    const int m = tok0 + tk, n = blockIdx.x * 64 + lr;
    uint32_t U = 0;
    for (int src = 0; src < S; ++src) U += (uint32_t)rbuf[(src * slots + slot) * 64 + lr];
    if (m < M && n < N) epilogue_store(p.e, m, n, U);
  }
}

template <int WB, int NT>
static cudaError_t launch_one(const MmaArgs& p, int split, size_t smem, cudaStream_t stream) {
  auto kern = gemm_mma_kernel<WB, NT>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.e.N + 63) / 64, (p.e.M + NT * 8 - 1) / (NT * 8), split);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = split;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p);
}

template <int WB>
static cudaError_t launch_wb(const MmaArgs& p, int nt, int split, size_t smem, cudaStream_t stream) {
  switch (nt) {
    case 1: return launch_one<WB, 1>(p, split, smem, stream);
    case 2: return launch_one<WB, 2>(p, split, smem, stream);
    case 4: return launch_one<WB, 4>(p, split, smem, stream);
    default: return launch_one<WB, 8>(p, split, smem, stream);
  }
}

size_t mma_smem_bytes(int bn, int split) {
  const size_t sb = (size_t)kKch * 8 * 4 * bn;                        // 32 bytes per word per token
  const size_t rb = (size_t)split * ((bn + split - 1) / split) * 64 * 4;  // reduction receive buffer
  return sb + rb;
}

cudaError_t launch_gemm_mma(const MmaArgs& p, int wbits, int bn, int split, cudaStream_t stream) {
  const int nt = bn / 8;
  const size_t smem = mma_smem_bytes(bn, split);
  switch (wbits) {
    case 1: return launch_wb<1>(p, nt, split, smem, stream);
    case 2: return launch_wb<2>(p, nt, split, smem, stream);
    case 3: return launch_wb<3>(p, nt, split, smem, stream);
    case 4: return launch_wb<4>(p, nt, split, smem, stream);
    case 5: return launch_wb<5>(p, nt, split, smem, stream);
    case 6: return launch_wb<6>(p, nt, split, smem, stream);
    case 7: return launch_wb<7>(p, nt, split, smem, stream);
    default: return launch_wb<8>(p, nt, split, smem, stream);
  }
}

}  // namespace apt
