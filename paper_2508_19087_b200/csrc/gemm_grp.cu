// gemm_grp.cu — grouped decode GEMM (apt_gemm_grouped): many independent APT W_p x A_q products with
// M <= 16 tokens each (a decoder layer's projections, the experts of a mixture-of-experts layer, the
// bench's 36 Llama-2-7B decode linears) in ONE persistent launch.
//
// Why: a single decode GEMM streams 2-23 MB of packed weights, i.e. 0.3-3.5 us at HBM speed, while a
// launch costs ~1 us of prologue and another ~1 us before its first weight bytes arrive
// (profiles/r2_dec_trace.txt, r2_chain_floor.json); chained, the per-GEMM kernels spend as much time
// ramping up and draining as streaming.  Here the CTAs of one grid split the SUM of all problems'
// weight blocks, so HBM never sees a launch boundary inside the group.
//
// Work decomposition (stream-K over the group): the unit is 128 weight rows x 256 K elements of one
// problem (problem-major, then 128-row tile, then K).  Units carry a cost (4 p_w + 2: the packed KB
// plus a fixed share for tokens and MMAs) and every CTA takes one contiguous range of equal total cost
// (midpoint rule, integer arithmetic: every CTA computes every other CTA's range without communication).
// A CTA accumulates consecutive units of a tile in registers; a tile covered by one CTA goes straight to
// the epilogue, a tile split between CTAs is reduced per 32-row warp slice: int32 partials
// ([worker][2][4 warps][16 x 32]) and an acq_rel ticket per slice, the last arrival adds and stores.
//
// CTA = 1 producer warp + 4 consumer warps.  The producer lane moves each unit into a ring slot with
// one cp.async.bulk per weight plane (4 KB: a 128-row x 256-K block of the tile-major layout is
// contiguous) and one 3-D TMA box of the activation digit view (2 x 8/16 rows x 128 bytes, 128B swizzle),
// completing on the slot's full mbarrier.  Consumer warp cw owns rows 32 cw .. 32 cw + 31 of the tile;
// lane (g, t) = (lane / 4, lane % 4) takes words t and t + 4 of the block for BOTH operands (so K
// agrees; conflict-free shared-memory reads), rebuilds the weight digits (rebuild_hi / rebuild_x16 /
// rebuild8: the shift half of the shift-add recovery) and issues mma.sync.m16n8k32 u8 with the
// weights as the B operand and tokens g, g + 8 as A (M > 8), or the weights as A (16 rows per MMA) and
// tokens g as B (M <= 8, half the MMAs); the epilogue is gemm_dec.cu's (rank-1 correction, scales,
// zero points, fp16 / int32, row / column layout; optionally also stored to peer buffers).  Group-wise
// scales use signed digits and s8 MMAs so that every 128-element group's product is exact on its own.
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

template <int WBMAX>
struct GrpShape {
  // CTA = 4 consumer warps (32 weight rows each) + 1 producer warp; unit = 128 weight rows x 256 K.
  // Slot = WBMAX weight planes of the unit (4 KB each: the tile-major [half][128 rows][4 words] block,
  // one contiguous bulk copy per plane) + the unit's token digits (one 3-D TMA box, 2 chunks x 8 / 16
  // rows x 128 bytes, zero fill past M, 128-byte swizzle: the fragment reads of rows g = 0..7 hit distinct banks).
  static constexpr int kTok = WBMAX * 4096;
  static constexpr int kSlot = WBMAX * 4096 + 4096;
#ifdef APT_GRP_D
  static constexpr int kD = APT_GRP_D;
#else
  static constexpr int kD = WBMAX <= 2 ? 4 : 2;  // 48 / 40 / 72 KB per CTA: 4 / 4 / 3 CTAs per SM
#endif
  static constexpr int kBarOff = kD * kSlot;
  // per consumer warp: the epilogue operands of its 32 rows / 16 tokens (w_rowsum, w_scale, a_rowsum,
  // a_scale: 384 bytes), copied in at the start of every segment so the epilogue never waits on global memory
  static constexpr int kEpiOff = (kBarOff + 2 * kD * 8 + 16 + 15) / 16 * 16;
  static constexpr int kSmem = kEpiOff + 4 * 384;
};

template <int WB>
__device__ __forceinline__ void grp_rebuild(const uint32_t* w, uint32_t (&o)[8]) {
  if constexpr (WB <= 2) rebuild_hi<WB>(w, o);
  else if constexpr (WB <= 4) rebuild_x16<WB>(w, o);
  else rebuild8<WB>(w, o);
}
// digits are u * 2^shift (gemm_dec.cu DecShape::kShift)
__device__ __forceinline__ int grp_shift(int wb) { return wb <= 2 ? 8 - wb : wb <= 4 ? 4 : 0; }

#ifdef APT_GRP_TRACE
// per-unit globaltimer timeline (profiling builds only): [cta][unit < 128][0 weights issued, 1 tokens
// issued, 2 consumer warp 0 saw full, 3 consumer warp 0 released]
__device__ unsigned long long g_grp_trace[1024][128][4];
__device__ __forceinline__ unsigned long long grp_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define GRP_TRACE(u, ph) do { if ((u) < 128 && blockIdx.x < 1024) g_grp_trace[blockIdx.x][(u)][(ph)] = grp_gtimer(); } while (0)
#else
#define GRP_TRACE(u, ph) do { } while (0)
#endif

__device__ __forceinline__ void grp_cp4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void grp_mma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void grp_mma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                           uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <bool S>
__device__ __forceinline__ void grp_mma_x(int* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
  if constexpr (S) grp_mma_s8(*reinterpret_cast<int(*)[4]>(c), a0, a1, a2, a3, b0, b1);
  else grp_mma(*reinterpret_cast<int(*)[4]>(c), a0, a1, a2, a3, b0, b1);
}

// Group-wise scales need every 128-element group's product on its own, so the digits become SIGNED
// (x * 2^s as int8: no rank-1 row-sum terms per group): bytewise d - h 2^s without borrows between bytes.
// Weight digits: top-aligned (W1, W2: u 2^(8-W); W4: u 16) and W8 -> flip bit 7; W3 (u 16 < 128) and
// W5-W7 (u < 2^W) -> ((d | 0x80) - h 2^s) ^ 0x80.
template <int WB>
__device__ __forceinline__ uint32_t grp_signed_w(uint32_t d) {
  if constexpr (WB <= 2 || WB == 4 || WB == 8) return d ^ 0x80808080u;
  else if constexpr (WB == 3) return ((d | 0x80808080u) - 0x40404040u) ^ 0x80808080u;
  else return ((d | 0x80808080u) - (1u << (WB - 1)) * 0x01010101u) ^ 0x80808080u;
}
// token digits u (low bits) -> signed codes x = u - h_a (hA = h_a * 0x01010101; h_a = 128 flips bit 7)
__device__ __forceinline__ uint32_t grp_signed_a(uint32_t u, uint32_t hA, bool ab8) {
  return ab8 ? u ^ 0x80808080u : ((u | 0x80808080u) - hA) ^ 0x80808080u;
}

// worker owning block i of problem q (midpoint rule): floor((2 cost0 + (2 i + 1) cost) * W / (2 T))
__device__ __forceinline__ int grp_owner(const GrpArgs& a, const GrpProblem& q, int64_t i) {
  return (int)((2 * q.cost0 + (2 * i + 1) * (int64_t)q.cost) * a.workers / (2 * a.total_cost));
}

// first block (problem p, local index i, global index gi) owned by a worker >= w; p = count if none
__device__ void grp_find(const GrpArgs& a, int w, int& p_out, int64_t& i_out, int64_t& g_out) {
  // the host computed every worker's first block with the same owner formula (apt.cu grp_run)
  const int64_t g = a.wstart[w];
  g_out = g;
  int p = 0;
  while (p + 1 < a.count && a.p[p + 1].blk0 <= g) ++p;
  if (g >= a.total_blocks) {
    p_out = a.count;
    i_out = 0;
    return;
  }
  p_out = p;
  i_out = g - a.p[p].blk0;
}

// one output element to out and, in launches with peers (a separate instantiation: even an untaken peer
// branch cost the epilogue-light decode launches 6%), to every peer buffer at the same offset (NEXT-4 ii)
template <bool PEERS, typename T>
__device__ __forceinline__ void grp_put(const GrpProblem& q, int64_t off, T v) {
  reinterpret_cast<T*>(q.e.out)[off] = v;
  if constexpr (PEERS)
    for (int j = 0; j < q.n_peers; ++j) reinterpret_cast<T*>(q.peers[j])[off] = v;
}

template <bool PEERS>
__device__ __forceinline__ void grp_store(const GrpProblem& q, const EpilogueArgs& e, int m, int n, uint32_t acc, int shift, int32_t ra,
                                          int32_t rw, float wsc, float as, float az = 0.f, float wz = 0.f,
                                          bool zp = false) {
  // acc = U * 2^shift; Y = U - h_w RA - h_a RW - Kpad h_a h_w (mod 2^32, exact: reading Q8)
  const uint32_t y = (acc >> shift) - (uint32_t)e.h_w * (uint32_t)ra - (uint32_t)e.h_a * (uint32_t)rw -
                     (uint32_t)e.kpad * (uint32_t)e.h_a * (uint32_t)e.h_w;
  if (m >= e.M || n >= e.N) return;
  const int64_t off = e.layout == 0 ? (int64_t)m * e.ldo + n : (int64_t)n * e.ldo + m;
  if (e.kind == 2) {
    float v = ((float)(int32_t)y * wsc) * as;
    if (zp) {  // zero points (P:199-201 on both operands): the apt_gemm zero-point formula, every operation
               // rounded on its own as in epilogue_zp.cu (bit-identical results)
      v = __fmul_rn(__fmul_rn((float)(int32_t)y, wsc), as);
      v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)rw, wsc), az));
      v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)ra, as), wz));
      v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)e.K, az), wz));
    }
    unsigned short hv;
    asm("cvt.rn.f16.f32 %0, %1;" : "=h"(hv) : "f"(v));
    grp_put<PEERS, unsigned short>(q, off, hv);
  } else {
    const uint32_t yb = 4u * y + 2u * (uint32_t)ra + 2u * (uint32_t)rw + (uint32_t)e.K;  // Y' (I2)
    grp_put<PEERS, int32_t>(q, off, (int32_t)(e.kind == 1 ? yb : y));
  }
}

// mbarrier phase wait: spin on try_wait (no suspend hint: the pipeline is short and a sleeping warp
// wakes late), or with the hint under APT_GRP_SLEEP
__device__ __forceinline__ void grp_wait(uint32_t bar, uint32_t parity) {
#ifdef APT_GRP_SLEEP
  mbar_wait(bar, parity);
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "GW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra GW_%=;\n}" ::"r"(bar), "r"(parity)
      : "memory");
#endif
}

#ifndef APT_GRP_MINB
#define APT_GRP_MINB 4  // four CTAs per SM (<= 102 registers): more consumer warps beat deeper rings (measured)
#endif
template <int WBMAX, bool MT1, bool GS, bool PEERS>
__global__ void __launch_bounds__(160, GS ? 2 : APT_GRP_MINB) gemm_grp_kernel(const __grid_constant__ GrpArgs a) {
  using SH = GrpShape<WBMAX>;
  constexpr int D = SH::kD;
  extern __shared__ __align__(1024) uint8_t smem[];  // no static shared memory: the swizzled token
  // (the token boxes need 1024-byte alignment)
  pdl_launch_dependents();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = blockIdx.x;  // worker = CTA
  const uint32_t sbase = smem_u32(smem);
  auto full = [&](int s) { return sbase + (uint32_t)(SH::kBarOff + s * 8); };
  auto empty = [&](int s) { return sbase + (uint32_t)(SH::kBarOff + (D + s) * 8); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  int p0, p1;
  int64_t i0, i1, gstart, gend;
  grp_find(a, w, p0, i0, gstart);
  grp_find(a, w + 1, p1, i1, gend);
  (void)p1;
  (void)i1;
  if (gstart >= gend) return;

#ifdef APT_GRP_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {  // the SM of the CTA (slot 127: beyond the traced units)
    unsigned sm_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
    g_grp_trace[blockIdx.x][127][3] = sm_ + 1;
  }
#endif
  if (warp == 4) {
    // ---- producer (one lane): per unit, WB bulk copies of 4 KB (weight planes) + M row copies of 256 B
    // (token digits), completing on the slot's full barrier; the weights of the first D units are
    // requested before griddepcontrol.wait (weights never depend on the previous kernel)
    if (lane != 0) return;
    // the current problem's fields live in registers (re-read from the parameter space only when the
    // producer moves on to the next problem: indexed constant loads are slow)
    int pp = p0, ptile = (int)(i0 / a.p[p0].nb), pblk = (int)(i0 - (int64_t)ptile * a.p[p0].nb);
    int pnb, ptiles, pwb;
    uint32_t ptx;
    int64_t pps;
    const uint32_t* pwp;
    const CUtensorMap* ptok;
    auto load_problem = [&]() {
      const GrpProblem& q = a.p[pp];
      pnb = q.nb;
      ptiles = q.tiles;
      pwb = q.wbits;
      pps = q.w_pstride;
      pwp = q.wp;
      ptok = &q.tok;
      ptx = (uint32_t)pwb * 4096u + 2u * (q.e.M <= 8 ? 8u : 16u) * 128u;  // (token rows >= M: the TMA zero fill)
    };
    load_problem();
    auto weights = [&](int slot) {
      mbar_expect_tx(full(slot), ptx);
      const uint32_t* src = pwp + ((int64_t)ptile * pnb + pblk) * 1024;
      for (int i = 0; i < pwb; ++i)
        bulk_load(sbase + (uint32_t)(slot * SH::kSlot + i * 4096), src + i * pps, 4096u, full(slot));
    };
    auto tokens = [&](int slot) {
      const uint32_t dst = sbase + (uint32_t)(slot * SH::kSlot + SH::kTok);
      tma_load_3d(dst, ptok, full(slot), 0, 0, pblk * 2);  // both 128-byte chunks of the block, one box
    };
    auto advance = [&]() {
      if (++pblk == pnb) {
        pblk = 0;
        if (++ptile == ptiles) {
          ptile = 0;
          if (++pp < a.count) load_problem();
        }
      }
    };
    const int64_t U = gend - gstart;
    const int pre = (int)min((int64_t)D, U);
    {
      const int qp = pp, qt = ptile, qb = pblk;
      for (int u = 0; u < pre; ++u) {
        weights(u);
        GRP_TRACE(u, 0);
        advance();
      }
      pdl_wait();
      pp = qp;
      ptile = qt;
      pblk = qb;
      load_problem();
      for (int u = 0; u < pre; ++u) {
        tokens(u);
        GRP_TRACE(u, 1);
        advance();
      }
    }
    int slot = pre % D;
    uint32_t ph = pre / D;  // completed passes over the ring
    for (int64_t u = pre; u < U; ++u) {
      grp_wait(empty(slot), (ph & 1) ^ 1);  // (the consumers fence their generic reads of the slot)
      weights(slot);
      GRP_TRACE(u, 0);
      tokens(slot);
      GRP_TRACE(u, 1);
      advance();
      if (++slot == D) {
        slot = 0;
        ++ph;
      }
    }
    return;
  }

  // ---- consumers: warp cw owns weight rows 32 cw .. 32 cw + 31 of each 128-row tile
  pdl_wait();  // scales / row sums of the activations, the output and the workspace
  const int cw = warp;
  const int g = lane >> 2, t = lane & 3;
  int cp = p0;
  int64_t ci = i0, cg = gstart;
  int slot = 0;
  uint32_t ph = 0;
  [[maybe_unused]] int tu = 0;  // units consumed (trace index)
#pragma unroll 1
  while (cg < gend) {
    const GrpProblem& q = a.p[cp];
    const int nb = q.nb;
    const int tile = (int)(ci / nb), b_in = (int)(ci - (int64_t)tile * nb);
    const int seg = (int)min((int64_t)(nb - b_in), gend - cg);
    const int n_w = tile * 128 + cw * 32;
    const bool narrow = MT1 && q.e.M <= 8;
    // lane (g, t) takes words t and t + 4 of every 256-element block (both operands, so K agrees):
    // tokens: row r, 32-byte word t of box 0 / box 1 = 16-byte chunks 2t, 2t + 1 at chunk ^ (r & 7)
    // (128-byte swizzle); weights: word t of half 0 / half 1 of row r = 4 bytes at h * 2048 + r * 16 + 4t.
    // Every 8-lane (16-byte) / 32-lane (4-byte) shared-memory access is conflict-free.  Token rows >= M
    // hold stale data; their products are never stored.
    const uint32_t trow0 = (uint32_t)(SH::kTok + g * 128);
    const uint32_t trow1 = trow0 + 8 * 128;
    // the token box is [2 chunks][R rows][128 bytes], R = 8 (M <= 8) or 16: chunk 1 starts R lines later
    // (a multiple of 8, so the 128-byte swizzle of line (chunk R + r) is r & 7 in both chunks)
    const uint32_t tbox = (q.e.M <= 8 ? 8u : 16u) * 128u;
    const uint32_t woff = (uint32_t)((cw * 32 + g) * 16 + t * 4);

    // epilogue operands of this segment's tile into the warp's area (asynchronous; waited for at the
    // epilogue): lane l -> row n_w + l, tokens l < 16
    const uint32_t epi_s = sbase + (uint32_t)(SH::kEpiOff + cw * 384);
    float* epi_p = reinterpret_cast<float*>(smem + SH::kEpiOff + cw * 384);
    if constexpr (!GS) {
      const int nl = min(n_w + lane, q.e.N - 1);
      grp_cp4(epi_s + lane * 4, q.e.w_rowsum + nl);
      if (q.e.kind == 2) grp_cp4(epi_s + 128 + lane * 4, q.e.w_scale + nl);
      if (lane < 16) {
        const int ml = min(lane, q.e.M - 1);
        grp_cp4(epi_s + 256 + lane * 4, q.e.a_rowsum + ml);
        if (q.e.kind == 2 && q.e.a_scale) grp_cp4(epi_s + 320 + lane * 4, q.e.a_scale + ml);
        else epi_p[80 + lane] = 1.f;
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }

    int acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0;
    // group-wise scales (GS): fp32 sums of the groups' scaled exact products (acc unused)
    float facc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) facc[j] = 0.f;
    const uint32_t hA = (uint32_t)q.e.h_a * 0x01010101u;
    const bool ab8 = q.e.h_a == 128;

    auto run = [&](auto wbc, auto mtc) {
      constexpr int WB = decltype(wbc)::value;
      constexpr int MT = decltype(mtc)::value;
      const int shift = grp_shift(WB);
#pragma unroll 1
      for (int b = 0; b < seg; ++b) {
        // GS: this block's two groups' scales (rows / tokens of the lane), requested before the wait
        [[maybe_unused]] float sw[2][8], sa[2][2];
        if constexpr (GS) {
          const int64_t g0 = 2 * (int64_t)(b_in + b);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              // MT 2: row n_w + 8 (j >> 1) + 2t + (j & 1); MT 1: row n_w + 16 (j >> 1) + g + 8 (j & 1) (j < 4)
              const int n = MT == 2 ? n_w + 8 * (j >> 1) + 2 * t + (j & 1) : n_w + 16 * (j >> 1) + g + 8 * (j & 1);
              sw[c][j] = (MT == 2 || j < 4) ? __ldg(q.w_gs + (g0 + c) * q.e.N + min(n, q.e.N - 1)) : 0.f;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int m = min(MT == 2 ? g + 8 * h : 2 * t + h, q.e.M - 1);
              sa[c][h] = q.a_gs ? __ldg(q.a_gs + (g0 + c) * q.a_gs_ld + m) : (q.e.a_scale ? __ldg(q.e.a_scale + m) : 1.f);
            }
          }
        }
        grp_wait(full(slot), ph & 1);
        if (cw == 0 && lane == 0) GRP_TRACE(tu, 2);
        const uint32_t sl = sbase + (uint32_t)(slot * SH::kSlot);
        uint4 tk0[4], tk1[4];  // [2 box + k]: word t (box 0) then word t + 4 (box 1), rows g / g + 8
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t ch = (uint32_t)((j >> 1) * tbox + (((2 * t + (j & 1)) ^ g) * 16));  // (line & 7) == g
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(tk0[j].x), "=r"(tk0[j].y), "=r"(tk0[j].z), "=r"(tk0[j].w)
                       : "r"(sl + trow0 + ch));
          if (MT == 2)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(tk1[j].x), "=r"(tk1[j].y), "=r"(tk1[j].z), "=r"(tk1[j].w)
                         : "r"(sl + trow1 + ch));
          if constexpr (GS) {
            uint32_t* t0 = reinterpret_cast<uint32_t*>(&tk0[j]);
            uint32_t* t1 = reinterpret_cast<uint32_t*>(&tk1[j]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              t0[e] = grp_signed_a(t0[e], hA, ab8);
              if (MT == 2) t1[e] = grp_signed_a(t1[e], hA, ab8);
            }
          }
        }
        int ai[2][16];  // GS: the block's per-group int products (c = group half)
        if constexpr (GS) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int j = 0; j < 16; ++j) ai[c][j] = 0;
        }
        if constexpr (MT == 2) {
          // weights = B operand (8 rows per MMA), tokens g, g + 8 = A operand: acc[4 qq + j]
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            uint2 wv[WB];  // .x = word t (half 0), .y = word t + 4 (half 1)
#pragma unroll
            for (int i = 0; i < WB; ++i) {
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv[i].x) : "r"(sl + woff + (uint32_t)(i * 4096 + qq * 128)));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wv[i].y) : "r"(sl + woff + (uint32_t)(i * 4096 + 2048 + qq * 128)));
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t wr[WB], o[8];
#pragma unroll
              for (int i = 0; i < WB; ++i) wr[i] = c ? wv[i].y : wv[i].x;
              grp_rebuild<WB>(wr, o);
              if constexpr (GS) {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = grp_signed_w<WB>(o[j]);
              }
              const uint32_t* ag = reinterpret_cast<const uint32_t*>(&tk0[2 * c]);
              const uint32_t* ah = reinterpret_cast<const uint32_t*>(&tk1[2 * c]);
              int* d = GS ? &ai[c][4 * qq] : &acc[4 * qq];
#pragma unroll
              for (int s4 = 0; s4 < 4; ++s4)
                grp_mma_x<GS>(d, ag[2 * s4], ah[2 * s4], ag[2 * s4 + 1], ah[2 * s4 + 1], o[2 * s4], o[2 * s4 + 1]);
            }
          }
        } else {
          // M <= 8: weights = A operand (rows g, g + 8 of each 16-row pair), tokens g = B operand: half the
          // MMAs; acc[4 P + j]
#pragma unroll
          for (int P = 0; P < 2; ++P) {
            uint2 wg[WB], wh[WB];
#pragma unroll
            for (int i = 0; i < WB; ++i) {
              const uint32_t bb = sl + woff + (uint32_t)(i * 4096 + P * 256);
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wg[i].x) : "r"(bb));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wg[i].y) : "r"(bb + 2048));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wh[i].x) : "r"(bb + 128));
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wh[i].y) : "r"(bb + 2048 + 128));
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t xg[WB], xh[WB], og[8], oh[8];
#pragma unroll
              for (int i = 0; i < WB; ++i) {
                xg[i] = c ? wg[i].y : wg[i].x;
                xh[i] = c ? wh[i].y : wh[i].x;
              }
              grp_rebuild<WB>(xg, og);
              grp_rebuild<WB>(xh, oh);
              if constexpr (GS) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  og[j] = grp_signed_w<WB>(og[j]);
                  oh[j] = grp_signed_w<WB>(oh[j]);
                }
              }
              const uint32_t* ag = reinterpret_cast<const uint32_t*>(&tk0[2 * c]);
              int* d = GS ? &ai[c][4 * P] : &acc[4 * P];
#pragma unroll
              for (int s4 = 0; s4 < 4; ++s4)
                grp_mma_x<GS>(d, og[2 * s4], oh[2 * s4], og[2 * s4 + 1], oh[2 * s4 + 1], ag[2 * s4], ag[2 * s4 + 1]);
            }
          }
        }
        // this warp is done with the slot: order its generic-proxy reads before the producer's next
        // async-proxy (bulk copy / TMA) write of the slot, then release it.  The fence sits here, not in
        // the producer: there it would also wait for the producer's own bulk copies in flight.
#ifndef APT_GRP_NOFENCE
        fence_proxy_async();
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(empty(slot));
        if (cw == 0 && lane == 0) GRP_TRACE(tu, 3);
        ++tu;
        if (++slot == D) {
          slot = 0;
          ++ph;
        }
        if constexpr (GS) {
          // fold the two groups: facc += ((float) Y_g * w_gscale) * a_gscale (Y_g exact: the int products
          // of signed digits, weights scaled by 2^shift)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int j = 0; j < (MT == 2 ? 16 : 8); ++j) {
              // MT 2: j = 4 qq + 2 h + cc (row 8 qq + 2t + cc, token g + 8h); MT 1: j = 4 P + 2 h + cc (row
              // 16 P + g + 8h, token 2t + cc)
              const float w_s = MT == 2 ? sw[c][2 * (j >> 2) + (j & 1)] : sw[c][2 * (j >> 2) + ((j >> 1) & 1)];
              const float a_s = MT == 2 ? sa[c][(j >> 1) & 1] : sa[c][j & 1];
              facc[j] += ((float)(ai[c][j] >> shift) * w_s) * a_s;
            }
        }
      }
      return 0;
    };
    auto run_w = [&](auto mtc) {
      using std::integral_constant;
      switch (q.wbits) {
        case 1: return run(integral_constant<int, 1>{}, mtc);
        case 2: return run(integral_constant<int, 2>{}, mtc);
        case 3: if constexpr (WBMAX >= 3) return run(integral_constant<int, 3>{}, mtc); break;
        case 4: if constexpr (WBMAX >= 4) return run(integral_constant<int, 4>{}, mtc); break;
        case 5: if constexpr (WBMAX >= 5) return run(integral_constant<int, 5>{}, mtc); break;
        case 6: if constexpr (WBMAX >= 6) return run(integral_constant<int, 6>{}, mtc); break;
        case 7: if constexpr (WBMAX >= 7) return run(integral_constant<int, 7>{}, mtc); break;
        default: if constexpr (WBMAX >= 8) return run(integral_constant<int, 8>{}, mtc); break;
      }
      return 0;
    };
    if (narrow) {
      if constexpr (MT1) run_w(std::integral_constant<int, 1>{});
    } else {
      run_w(std::integral_constant<int, 2>{});
    }
    const int shift = grp_shift(q.wbits);
    if constexpr (GS) {  // the split-tile exchange below moves the fp32 sums as their bit patterns
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = __float_as_int(facc[j]);
    }

    // ---- the tile: whole (one CTA) or split (partials + ticket; the last CTA to arrive reduces)
    // a tile this segment covers whole needs no owner lookup; a split tile finds its first / last owner
    // in the range table (binary search over indexed parameter loads: only for split tiles)
    const bool whole = b_in == 0 && seg == nb;
    const int64_t tfirst = (int64_t)tile * nb;
    const int fw = whole ? w : grp_owner(a, q, tfirst), lw = whole ? w : grp_owner(a, q, tfirst + nb - 1);
    bool epi = true;
    if (fw != lw) {
      // each consumer warp reduces its own 32-row slice: partial, warp barrier (orders the lanes' stores
      // before lane 0's ticket), acq_rel ticket at GPU scope (release: cumulative over those stores;
      // acquire: the last arrival sees every other CTA's slice), warp barrier, reduction
      int* part = a.partials + (((int64_t)w * 2 + (w == fw ? 1 : 0)) * 4 + cw) * 512;
#pragma unroll
      for (int j = 0; j < 16; ++j) __stcg(part + j * 32 + lane, acc[j]);
      __syncwarp();
      unsigned prev = 0;
      if (lane == 0) {
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.tickets + fw * 4 + cw) : "memory");
        if (prev == (unsigned)(lw - fw))
          asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(a.tickets + fw * 4 + cw), "r"(0u) : "memory");
      }
      prev = __shfl_sync(0xffffffffu, prev, 0);
      epi = prev == (unsigned)(lw - fw);
      if (epi) {
        __syncwarp();
        // int32 partials add exactly in any order; the fp32 group-scale sums are added in worker order
        // (this warp's own slice re-read from memory in its place), so the rounding does not depend on
        // which CTA happened to arrive last
        if constexpr (GS) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = __float_as_int(0.f);
        }
#pragma unroll 1
        for (int o = fw; o <= lw; ++o) {
          if (!GS && o == w) continue;
          const int* po = a.partials + (((int64_t)o * 2 + (o == fw ? 1 : 0)) * 4 + cw) * 512;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int v = __ldcg(po + j * 32 + lane);
            acc[j] = GS ? __float_as_int(__int_as_float(acc[j]) + __int_as_float(v)) : acc[j] + v;
          }
        }
      }
    }
    if (epi && GS) {
      // group-wise scales: out = RN_fp16(sum_g ((float) Y_g * w_gscale) * a_gscale), fp16 row / column layout
      const EpilogueArgs& e = q.e;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int m = narrow ? 2 * t + (j & 1) : g + 8 * ((j >> 1) & 1);
        const int n = narrow ? n_w + 16 * (j >> 2) + g + 8 * ((j >> 1) & 1) : n_w + 8 * (j >> 2) + 2 * t + (j & 1);
        if ((narrow && j >= 8) || m >= e.M || n >= e.N) continue;
        unsigned short hv;
        asm("cvt.rn.f16.f32 %0, %1;" : "=h"(hv) : "f"(__int_as_float(acc[j])));
        grp_put<PEERS, unsigned short>(q, e.layout == 0 ? (int64_t)m * e.ldo + n : (int64_t)n * e.ldo + m, hv);
      }
    } else if (epi) {
      const EpilogueArgs& e = q.e;
      const bool f16 = e.kind == 2;
      const bool zp = f16 && (q.w_zero || q.a_zero);
      // the segment's prefetched operands: rows [0, 32) at 0 / 128 (int / float), tokens at 256 / 320
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncwarp();
      const int32_t* ep_rw = reinterpret_cast<const int32_t*>(epi_p);
      const int32_t* ep_ra = reinterpret_cast<const int32_t*>(epi_p + 64);
      if (!narrow) {  // acc[4 qq + 2 h + c]: token g + 8h, weight row n_w + 8 qq + 2t + c
        int32_t ra[2];
        float as[2], az[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = min(g + 8 * h, e.M - 1);
          ra[h] = ep_ra[g + 8 * h];
          as[h] = epi_p[80 + g + 8 * h];
          az[h] = (zp && q.a_zero) ? __ldg(q.a_zero + m) : 0.f;
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int n = n_w + 8 * qq + 2 * t + c, nc = min(n, e.N - 1);
            const int32_t rw = ep_rw[8 * qq + 2 * t + c];
            const float wsc = f16 ? epi_p[32 + 8 * qq + 2 * t + c] : 0.f;
            const float wz = (zp && q.w_zero) ? __ldg(q.w_zero + nc) : 0.f;
#pragma unroll
            for (int h = 0; h < 2; ++h)
              grp_store<PEERS>(q, e, g + 8 * h, n, (uint32_t)acc[4 * qq + 2 * h + c], shift, ra[h], rw, wsc, as[h], az[h], wz, zp);
          }
      } else {  // acc[4 P + 2 h + c]: weight row n_w + 16 P + g + 8 h, token 2t + c
        int32_t ra[2];
        float as[2], az[2];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int m = min(2 * t + c, e.M - 1);
          ra[c] = ep_ra[2 * t + c];
          as[c] = epi_p[80 + 2 * t + c];
          az[c] = (zp && q.a_zero) ? __ldg(q.a_zero + m) : 0.f;
        }
#pragma unroll
        for (int P = 0; P < 2; ++P)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int n = n_w + 16 * P + g + 8 * h, nc = min(n, e.N - 1);
            const int32_t rw = ep_rw[16 * P + g + 8 * h];
            const float wsc = f16 ? epi_p[32 + 16 * P + g + 8 * h] : 0.f;
            const float wz = (zp && q.w_zero) ? __ldg(q.w_zero + nc) : 0.f;
#pragma unroll
            for (int c = 0; c < 2; ++c)
              grp_store<PEERS>(q, e, 2 * t + c, n, (uint32_t)acc[4 * P + 2 * h + c], shift, ra[c], rw, wsc, as[c], az[c], wz, zp);
          }
      }
    }
    ci += seg;
    cg += seg;
    if (ci == (int64_t)q.tiles * nb) {
      ci = 0;
      ++cp;
    }
  }
}

#ifndef APT_GRP_MT1
#define APT_GRP_MT1 true
#endif

template <int WBMAX, bool MT1, bool GS, bool PEERS>
static cudaError_t launch_grp2(const GrpArgs& a, int ctas, cudaStream_t stream) {
  constexpr int kSmem = GrpShape<WBMAX>::kSmem;
  cudaError_t err = set_smem_once<gemm_grp_kernel<WBMAX, MT1, GS, PEERS>>(kSmem);
  if (err != cudaSuccess) return err;
  return launch_pdl(gemm_grp_kernel<WBMAX, MT1, GS, PEERS>, dim3(ctas), dim3(160), kSmem, stream, dim3(1, 1, 1), a);
}

template <bool PEERS>
static cudaError_t launch_grp1(const GrpArgs& a, int cls, bool gs, int ctas, cudaStream_t stream) {
  switch (cls * 2 + (gs ? 1 : 0)) {
    case 4: return launch_grp2<2, APT_GRP_MT1, false, PEERS>(a, ctas, stream);
    case 5: return launch_grp2<2, APT_GRP_MT1, true, PEERS>(a, ctas, stream);
    case 8: return launch_grp2<4, APT_GRP_MT1, false, PEERS>(a, ctas, stream);
    case 9: return launch_grp2<4, APT_GRP_MT1, true, PEERS>(a, ctas, stream);
    case 17: return launch_grp2<8, APT_GRP_MT1, true, PEERS>(a, ctas, stream);
    default: return launch_grp2<8, APT_GRP_MT1, false, PEERS>(a, ctas, stream);
  }
}

int grp_wbmax_class(int wbmax) { return wbmax <= 2 ? 2 : wbmax <= 4 ? 4 : 8; }
// CTAs per SM (shared memory 48 / 40 / 72 KB per CTA at WBMAX 2 / 4 / 8; registers: <= 102 per thread
// for four CTAs; the group-scale path needs more registers: two)
int grp_ctas_per_sm(int wbmax, bool gs) { return gs ? 2 : grp_wbmax_class(wbmax) <= 4 ? 4 : 3; }

cudaError_t launch_gemm_grp(const GrpArgs& a, int wbmax, int ctas, bool gs, bool peers, cudaStream_t stream) {
  const int cls = grp_wbmax_class(wbmax);
  return peers ? launch_grp1<true>(a, cls, gs, ctas, stream) : launch_grp1<false>(a, cls, gs, ctas, stream);
}

}  // namespace apt

#ifdef APT_GRP_TRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_grp_trace(unsigned long long* host, int reset) {
  if (reset) {
    static unsigned long long zero[1024 * 128 * 4];
    return (int)cudaMemcpyToSymbol(apt::g_grp_trace, zero, sizeof(zero));
  }
  return (int)cudaMemcpyFromSymbol(host, apt::g_grp_trace, sizeof(unsigned long long) * 1024 * 128 * 4);
}
#endif
