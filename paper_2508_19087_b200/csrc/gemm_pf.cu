// gemm_pf.cu — persistent tcgen05 GEMM for token-rich shapes (M > 64: prefill, Llama-3-70B, the sweep).
//
// Why (DESIGN.md §7 "Prefill"): the non-persistent tile (gemm_tc.cu) pays ~2.5 us of setup and pipeline
// fill and ~4 us of epilogue per 128 x 256 tile with the tensor pipe idle, and 256 tiles of a 4096^2
// prefill GEMM are 1.73 waves on 148 SMs.  Here one CTA per SM walks the tile list (tile t, t + grid, ...)
// with every ring running continuously across tiles, and the accumulator is double-buffered in TMEM, so
// the epilogue of tile i (dedicated warps) overlaps the MMAs of tile i + 1.
//
// CTA = 32 * (8 + 4 kConvPar) threads, tile = 128 weight rows x 128 / 192 / 256 tokens:
//   warp 0      producer (one thread): weight chunks (256 K elements of the tile's 128 rows, every plane: a
//               4 KB bulk copy per plane in the tile-major layout, one 3-D TMA box otherwise) into a slot
//               ring — requested before griddepcontrol.wait for the first tiles, weights never depend on
//               the previous kernel — and the token digits (128-byte swizzled TMA boxes) into a stage ring;
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma (kind::i8 K=32, or kind::mxf4 K=64) per step into
//               accumulator buffer (tile & 1); waits until the epilogue released that buffer;
//   warp 2      TMEM allocation (512 columns: 2 x 128 accumulator, 4 x 32 A ring, 32 mxf4 scale columns);
//   warps 4..    converters (kConvPar per TMEM sub-partition, taking turns by step): planes -> digits
//               (rebuild8, or rebuild_e2m1 for mxf4) -> tcgen05.st into the A ring;
//   last 4 warps epilogue (thread = weight row = TMEM lane): tcgen05.ld of the finished buffer, rank-1
//               corrections and scales (common.cuh arithmetic), stores; then release the buffer.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"
#include "tc_ptx.cuh"

namespace apt {

constexpr int kPfBM = 128;  // weight rows per tile (MMA M)
#ifndef APT_PF256_AS
#define APT_PF256_AS 2  // shared-memory A stages of the 256-token tile
#endif
// converter warps per TMEM sub-partition (steps alternate between them): one at wbits <= 4 (fewer warps
// contending for shared memory and issue slots: 1-5% faster on the 192 / 256-token tiles), two at
// wbits > 4 (the 8-plane rebuild needs the second warp's latency hiding: W8A8 4096^3 73.5 vs 77.1 us).
// EP = epilogue warps per sub-partition (each drains 1 / EP of the tile's token columns): 2 for short
// walks (<= 8 tiles per CTA, where the last tile's exposed epilogue matters: 3-6% on the prefill shapes),
// 1 for long ones (the extra warps cost 3% over the 25-tile Llama-3-70B walk)
template <int WB, int EP>
struct PfWarps {
  static constexpr int kConvPar = WB <= 4 ? 1 : 2;
  static constexpr int kEpiWarp0 = 4 + 4 * kConvPar;  // first epilogue warp
  static constexpr int kThreads = 32 * (kEpiWarp0 + 4 * EP);
};

// BN = tokens per tile (MMA N): 128; 192 (i8 only) — 2 x 192 accumulator columns + the 4 x 32 A ring fill
// the 512 TMEM columns; 256 (i8 only) — the two accumulators take all 512 columns, so the converters
// write the rebuilt weight digits to a shared-memory A ring (128-byte swizzled K-major rows, the layout
// the token TMA boxes have) and the MMAs read both operands through descriptors
template <int WB, bool MX, int BN>
struct PfSmem {
  static constexpr bool kASmem = BN == 256;
  static constexpr int kBBytes = BN * 128;  // token bytes per step: 128 rows x 128 B (i8 128 K / mxf4 256 K)
  static constexpr int kWChunk = WB * 4096;    // weight bytes per 256-K chunk, every plane
  static constexpr int kWSlots = kASmem ? (WB <= 2 ? 4 : WB <= 4 ? 3 : 2) : (WB <= 2 ? 8 : WB <= 4 ? 6 : 3);
  static constexpr int kAStages = kASmem ? APT_PF256_AS : 4;
  static constexpr int kABytes = kPfBM * 128;  // one A stage in shared memory: 128 rows x 128 K bytes
  // 256-token tiles: as many token stages as the rest of the 227 KB leaves (the token ring hides the L2
  // latency of the 32 KB boxes; 3 stages starve the MMAs)
  static constexpr int kTokFit = (225 * 1024 - kAStages * kABytes - kWSlots * kWChunk) / kBBytes;
  static constexpr int kTokStages = BN <= 128 ? 6 : BN <= 192 ? 4 : (kTokFit < 6 ? kTokFit : 6);
  static constexpr int kBOff = 0;
  static constexpr int kWOff = kTokStages * kBBytes;
  static constexpr int kAOff = kWOff + kWSlots * kWChunk;
  static constexpr int kBarOff = kAOff + (kASmem ? kAStages * kABytes : 0);
  static constexpr int kNumBars = 2 * kTokStages + 2 * kWSlots + 2 * kAStages + 4;
  static constexpr int kTotal = kBarOff + kNumBars * 8 + 16 + 1024;  // + TMEM slot + alignment slack
};

template <int WB, bool MX, int BN, int EP>
__global__ void __launch_bounds__(PfWarps<WB, EP>::kThreads, 1) gemm_pf_kernel(const __grid_constant__ CUtensorMap tm_w,
                                                               const __grid_constant__ CUtensorMap tm_b, TcArgs p) {
  static_assert(BN == 128 || ((BN == 192 || BN == 256) && !MX), "token tile");
  using L = PfSmem<WB, MX, BN>;
  constexpr int ST = L::kTokStages, WS = L::kWSlots, AS = L::kAStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sB = base + L::kBOff, sW = base + L::kWOff, bars = base + L::kBarOff;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (ST + s); };
  auto wfull = [&](int c) { return bars + 8u * (2 * ST + c); };
  auto wempty = [&](int c) { return bars + 8u * (2 * ST + WS + c); };
  auto a_full = [&](int a) { return bars + 8u * (2 * ST + 2 * WS + a); };
  auto a_empty = [&](int a) { return bars + 8u * (2 * ST + 2 * WS + AS + a); };
  auto acc_full = [&](int b) { return bars + 8u * (2 * ST + 2 * WS + 2 * AS + b); };
  auto acc_empty = [&](int b) { return bars + 8u * (2 * ST + 2 * WS + 2 * AS + 2 + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L::kBarOff + L::kNumBars * 8);
  constexpr uint32_t kAcol0 = 2 * BN;         // A ring after the two accumulator buffers
  constexpr uint32_t kScol0 = kAcol0 + 32 * AS;  // mxf4 unit scale factors
  constexpr int kShift = MX ? 0 : WB <= 2 ? 8 - WB : WB <= 4 ? 4 : 0;  // i8 weight digits are u * 2^kShift
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int tiles_n = (p.e.N + kPfBM - 1) / kPfBM, tiles_m = (p.e.M + BN - 1) / BN;
  const int tiles = tiles_n * tiles_m;
  const int chunks = p.k_words >> 3;                  // 256-element weight chunks per tile
  const int nsteps = MX ? chunks : 2 * chunks;         // MMA steps per tile
  const bool tiled = p.w_tiled != 0;
  pdl_launch_dependents();

  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int c = 0; c < WS; ++c) {
      mbar_init(wfull(c), 1);
      mbar_init(wempty(c), MX ? 4 : 8);  // the converter warps reading the chunk (two steps of two parities, i8)
    }
    for (int a = 0; a < AS; ++a) {
      mbar_init(a_full(a), 4);  // the four converter warps of one parity (one per TMEM sub-partition)
      mbar_init(a_empty(a), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full(b), 1);
      mbar_init(acc_empty(b), 4 * EP);  // the epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int gc = 0, gs = 0;  // global weight-chunk and token-step counters (ring positions)
      bool waited = false;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int tn = t / tiles_m, tm = t % tiles_m;
        const uint32_t* wtile = p.wp + (int64_t)tn * (p.k_words >> 3) * 1024;
        for (int c = 0; c < chunks; ++c, ++gc) {
          const int slot = gc % WS;
          mbar_wait(wempty(slot), ((gc / WS) & 1) ^ 1);
          // the converters' generic-proxy reads of this slot (released through wempty) before the async-proxy
          // (bulk copy / TMA) overwrite: a proxy fence makes the write-after-read order explicit
          fence_proxy_async();
          mbar_expect_tx(wfull(slot), (uint32_t)L::kWChunk);
          if (tiled) {
#pragma unroll
            for (int i = 0; i < WB; ++i)
              bulk_load(sW + slot * L::kWChunk + i * 4096, wtile + (int64_t)i * p.w_pstride + (int64_t)c * 1024, 4096u,
                        wfull(slot));
          } else {
            tma_load_3d(sW + slot * L::kWChunk, &tm_w, wfull(slot), c * 8, tn * kPfBM, 0);
          }
          if (!waited) {  // the token digits may come from the previous kernel
            pdl_wait();
            waited = true;
          }
          for (int h = 0; h < (MX ? 1 : 2); ++h, ++gs) {
            const int s = gs % ST;
            mbar_wait(empty(s), ((gs / ST) & 1) ^ 1);
            mbar_expect_tx(full(s), (uint32_t)L::kBBytes);
            tma_load_2d(sB + s * L::kBBytes, &tm_b, full(s), (MX ? c : 2 * c + h) * 128, tm * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = MX ? ((1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | (1u << 23) |
                                       ((uint32_t)(kPfBM >> 4) << 24))
                                    : ((2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(kPfBM >> 4) << 24));
      int gs = 0, li = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++li) {
        const int buf = li & 1;
        mbar_wait(acc_empty(buf), ((li >> 1) & 1) ^ 1);  // the epilogue of tile li - 2 released it
        tc_fence_after();
        const uint32_t dcol = tmem + (uint32_t)(buf * BN);
        for (int j = 0; j < nsteps; ++j, ++gs) {
          const int s = gs % ST, a = gs % AS;
          mbar_wait(full(s), (gs / ST) & 1);
          mbar_wait(a_full(a), (gs / AS) & 1);
          tc_fence_after();
          const uint64_t bdesc = umma_desc_sw128(sB + s * L::kBBytes);
          const uint64_t adesc = umma_desc_sw128(base + L::kAOff + a * L::kABytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if constexpr (L::kASmem)
              tc_mma_i8_ss(dcol, adesc + (uint64_t)(2 * kk), bdesc + (uint64_t)(2 * kk), idesc, (j | kk) != 0);
            else if constexpr (MX)
              tc_mma_mxf4(dcol, tmem + kAcol0 + 32 * a + 8 * kk, bdesc + (uint64_t)(2 * kk), idesc, (j | kk) != 0,
                          tmem + kScol0, tmem + kScol0 + 16);
            else
              tc_mma_i8(dcol, tmem + kAcol0 + 32 * a + 8 * kk, bdesc + (uint64_t)(2 * kk), idesc, (j | kk) != 0);
          }
          tc_commit(empty(s));
          tc_commit(a_empty(a));
        }
        tc_commit(acc_full(buf));
      }
    }
  } else if (warp >= 4 && warp < PfWarps<WB, EP>::kEpiWarp0) {
    // ------------------------------------------------------------ converters
    const int cw = warp - 4, sub = cw & 3, par = cw >> 2;
    const int r = sub * 32 + lane;
    const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
    if constexpr (MX) {
      if (par == 0) {
        uint32_t one[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) one[i] = 0x7F7F7F7Fu;
        tmem_st32<32>(tmem + lane_off + kScol0, one);
      }
    }
    const uint8_t* wsm = gbase + L::kWOff;
    int total = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) total += nsteps;
    for (int gs = par; gs < total; gs += PfWarps<WB, EP>::kConvPar) {
      const int gc = MX ? gs : gs >> 1, q = MX ? 0 : gs & 1;
      const int slot = gc % WS;
      mbar_wait(wfull(slot), (gc / WS) & 1);
      constexpr int kH = MX ? 2 : 1;
      uint4 v[kH][WB];
#pragma unroll
      for (int h = 0; h < kH; ++h)
#pragma unroll
        for (int i = 0; i < WB; ++i) {
          const int qq = MX ? h : q;
          // tile-major: [plane][half][row][4 words]; 3-D TMA box: [plane][row][8 words]
          v[h][i] = *reinterpret_cast<const uint4*>(wsm + slot * L::kWChunk + i * 4096 +
                                                    (tiled ? qq * 2048 + r * 16 : (r * 8 + 4 * qq) * 4));
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(wempty(slot));
      uint32_t d[32];
      if constexpr (MX) {
#pragma unroll
        for (int wi = 0; wi < 8; ++wi) {
          uint32_t w[3] = {0u, 0u, 0u}, g[4];
#pragma unroll
          for (int i = 0; i < WB; ++i) {
            const uint4& tt = v[wi >> 2][i];
            const int jj = wi & 3;
            w[i] = jj == 0 ? tt.x : jj == 1 ? tt.y : jj == 2 ? tt.z : tt.w;
          }
          rebuild_e2m1<(WB <= 3 ? WB : 3)>(w, g);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) d[4 * wi + cc] = g[cc];
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t w[WB], o[8];
#pragma unroll
          for (int i = 0; i < WB; ++i) w[i] = jj == 0 ? v[0][i].x : jj == 1 ? v[0][i].y : jj == 2 ? v[0][i].z : v[0][i].w;
          // scaled digits u * 2^kShift (rebuild_hi / rebuild_x16): fewer integer-ALU ops per element, the
          // converters' bound at 128-token tiles; the epilogue shifts the exact sum back (reading R-DEC)
          if constexpr (WB <= 2) rebuild_hi<WB>(w, o);
          else if constexpr (WB <= 4) rebuild_x16<WB>(w, o);
          else rebuild8<WB>(w, o);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) d[8 * jj + cc] = o[cc];
        }
      }
      const int a = gs % AS;
      mbar_wait(a_empty(a), ((gs / AS) & 1) ^ 1);
      if constexpr (L::kASmem) {
        // row r of the stage: 16-byte chunk c (TMEM columns 4c .. 4c + 3, K bytes 16c ..) at chunk c ^ (r % 8)
        uint8_t* arow = gbase + L::kAOff + a * L::kABytes + r * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(arow + ((c ^ (r & 7)) << 4)) = make_uint4(d[4 * c], d[4 * c + 1], d[4 * c + 2], d[4 * c + 3]);
        fence_proxy_async();  // the generic-proxy stores, before the MMA's async-proxy reads
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(a));
      } else {
        tc_fence_after();
        tmem_st32<32>(tmem + lane_off + kAcol0 + 32 * a, d);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(a));
      }
    }
  } else if (warp >= PfWarps<WB, EP>::kEpiWarp0) {
    // ------------------------------------------------------------ epilogue
    const int ew = (warp - PfWarps<WB, EP>::kEpiWarp0) & 3;  // == warp % 4: this warp's TMEM sub-partition
    const int eh = (warp - PfWarps<WB, EP>::kEpiWarp0) >> 2;  // which 1 / EP of the tile's token columns
    const int r = ew * 32 + lane;
    const uint32_t lane_off = (uint32_t)(ew * 32) << 16;
    pdl_wait();  // token row sums / scales and the output may be touched by the previous kernel
    const bool vec_tok = p.e.a_scale && ((reinterpret_cast<uintptr_t>(p.e.a_rowsum) | reinterpret_cast<uintptr_t>(p.e.a_scale)) & 15u) == 0;
    int li = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++li) {
      const int buf = li & 1;
      const int tn = t / tiles_m, tm = t % tiles_m;
      const int n = tn * kPfBM + r, m0 = tm * BN;
      const int nc = min(n, p.e.N - 1);
      const int32_t rw = __ldg(p.e.w_rowsum + nc);
      const float wsc = p.e.kind == 2 ? __ldg(p.e.w_scale + nc) : 0.f;
      const uint32_t cn = (uint32_t)p.e.h_a * (uint32_t)rw + (uint32_t)p.e.kpad * (uint32_t)p.e.h_a * (uint32_t)p.e.h_w;
      mbar_wait(acc_full(buf), (li >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = eh * (BN / EP); c0 < (eh + 1) * (BN / EP); c0 += 32) {
        uint32_t acc[32];
        tmem_ld32(tmem + lane_off + (uint32_t)(buf * BN + c0), acc);
        if constexpr (MX) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) acc[jj] = (uint32_t)__float2int_rn(__uint_as_float(acc[jj]));
        } else if constexpr (kShift > 0) {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) acc[jj] >>= kShift;
        }
        const int mb = m0 + c0;
        if (n >= p.e.N || mb >= p.e.M) {
          // nothing of this chunk is stored by this lane
        } else if (p.e.kind == 2) {
          uint32_t hv[16];
          if (vec_tok && mb + 32 <= p.e.M) {
            // the chunk's 32 token row sums / scales as 16-byte loads (same values for every lane)
#pragma unroll
            for (int j4 = 0; j4 < 32; j4 += 4) {
              const int4 ra4 = __ldg(reinterpret_cast<const int4*>(p.e.a_rowsum + mb + j4));
              const float4 as4 = __ldg(reinterpret_cast<const float4*>(p.e.a_scale + mb + j4));
              const int32_t rr[4] = {ra4.x, ra4.y, ra4.z, ra4.w};
              const float aa[4] = {as4.x, as4.y, as4.z, as4.w};
              float v4[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t y = acc[j4 + e] - (uint32_t)p.e.h_w * (uint32_t)rr[e] - cn;
                v4[e] = ((float)(int32_t)y * wsc) * aa[e];
              }
              hv[j4 / 2] = pack_f16x2(v4[0], v4[1]);
              hv[j4 / 2 + 1] = pack_f16x2(v4[2], v4[3]);
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 32; jj += 2) {
              float v2[2];
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) {
                const int m = min(mb + jj + e2, p.e.M - 1);
                const uint32_t y = acc[jj + e2] - (uint32_t)p.e.h_w * (uint32_t)__ldg(p.e.a_rowsum + m) - cn;
                v2[e2] = ((float)(int32_t)y * wsc) * (p.e.a_scale ? __ldg(p.e.a_scale + m) : 1.f);
              }
              hv[jj / 2] = pack_f16x2(v2[0], v2[1]);
            }
          }
          unsigned short* outh = reinterpret_cast<unsigned short*>(p.e.out);
          if (p.e.layout == 0) {
            unsigned short* qp = outh + (int64_t)mb * p.e.ldo + n;
#pragma unroll
            for (int jj = 0; jj < 32; ++jj)
              if (mb + jj < p.e.M) qp[(int64_t)jj * p.e.ldo] = (unsigned short)(hv[jj / 2] >> (16 * (jj & 1)));
          } else {
            unsigned short* qp = outh + (int64_t)n * p.e.ldo + mb;
            if (mb + 32 <= p.e.M && ((reinterpret_cast<uintptr_t>(qp) & 15u) == 0)) {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 8)
                *reinterpret_cast<uint4*>(qp + jj) = make_uint4(hv[jj / 2], hv[jj / 2 + 1], hv[jj / 2 + 2], hv[jj / 2 + 3]);
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj)
                if (mb + jj < p.e.M) qp[jj] = (unsigned short)(hv[jj / 2] >> (16 * (jj & 1)));
            }
          }
        } else {
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int m = mb + jj;
            if (m < p.e.M)
              epilogue_store_v(p.e, m, n, acc[jj], __ldg(p.e.a_rowsum + m), rw, wsc,
                               (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty(buf));
    }
  }
  tc_fence_before();
  __syncwarp();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

template <int WB, bool MX, int BN, int EP>
static cudaError_t launch_pf3(const CUtensorMap& tw, const CUtensorMap& tb, const TcArgs& p, int grid, cudaStream_t stream) {
  using L = PfSmem<WB, MX, BN>;
  static_assert(L::kTotal <= 227 * 1024, "shared memory budget");
  cudaError_t err = set_smem_once<gemm_pf_kernel<WB, MX, BN, EP>>(L::kTotal);
  if (err != cudaSuccess) return err;
  return launch_pdl(gemm_pf_kernel<WB, MX, BN, EP>, dim3(grid), dim3(PfWarps<WB, EP>::kThreads), L::kTotal, stream,
                    dim3(1, 1, 1), tw, tb, p);
}

template <int WB, bool MX, int BN>
static cudaError_t launch_pf2(const CUtensorMap& tw, const CUtensorMap& tb, const TcArgs& p, cudaStream_t stream) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = ((p.e.N + kPfBM - 1) / kPfBM) * ((p.e.M + BN - 1) / BN);
  const int grid = tiles < sms ? tiles : sms;
  if constexpr (BN == 256) {
    if ((tiles + grid - 1) / grid <= 8) return launch_pf3<WB, MX, BN, 2>(tw, tb, p, grid, stream);
  }
  return launch_pf3<WB, MX, BN, 1>(tw, tb, p, grid, stream);
}

cudaError_t launch_gemm_pf(const TcArgs& p, int wbits, int mx, int bn, cudaStream_t stream) {
  if (bn != 128 && ((bn != 192 && bn != 256) || mx)) return cudaErrorInvalidValue;
  PFN_encodeTiled_t enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tw, tb;
  if (!make_plane_map(&tw, p.wp, p.k_words, p.e.N, wbits, 8, kPfBM)) return cudaErrorInvalidValue;
  {
    const cuuint64_t kp = (cuuint64_t)p.k_words * (mx ? 16 : 32);
    cuuint64_t dims[2] = {kp, (cuuint64_t)p.e.M};
    cuuint64_t strides[1] = {kp};
    cuuint32_t box[2] = {128u, (cuuint32_t)bn};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p.adig), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  if (mx) {
    switch (wbits) {
      case 1: return launch_pf2<1, true, 128>(tw, tb, p, stream);
      case 2: return launch_pf2<2, true, 128>(tw, tb, p, stream);
      case 3: return launch_pf2<3, true, 128>(tw, tb, p, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  if (bn == 256) {
    switch (wbits) {
      case 1: return launch_pf2<1, false, 256>(tw, tb, p, stream);
      case 2: return launch_pf2<2, false, 256>(tw, tb, p, stream);
      case 3: return launch_pf2<3, false, 256>(tw, tb, p, stream);
      case 4: return launch_pf2<4, false, 256>(tw, tb, p, stream);
      case 5: return launch_pf2<5, false, 256>(tw, tb, p, stream);
      case 6: return launch_pf2<6, false, 256>(tw, tb, p, stream);
      case 7: return launch_pf2<7, false, 256>(tw, tb, p, stream);
      default: return launch_pf2<8, false, 256>(tw, tb, p, stream);
    }
  }
  if (bn == 192) {
    switch (wbits) {
      case 1: return launch_pf2<1, false, 192>(tw, tb, p, stream);
      case 2: return launch_pf2<2, false, 192>(tw, tb, p, stream);
      case 3: return launch_pf2<3, false, 192>(tw, tb, p, stream);
      case 4: return launch_pf2<4, false, 192>(tw, tb, p, stream);
      case 5: return launch_pf2<5, false, 192>(tw, tb, p, stream);
      case 6: return launch_pf2<6, false, 192>(tw, tb, p, stream);
      case 7: return launch_pf2<7, false, 192>(tw, tb, p, stream);
      default: return launch_pf2<8, false, 192>(tw, tb, p, stream);
    }
  }
  switch (wbits) {
    case 1: return launch_pf2<1, false, 128>(tw, tb, p, stream);
    case 2: return launch_pf2<2, false, 128>(tw, tb, p, stream);
    case 3: return launch_pf2<3, false, 128>(tw, tb, p, stream);
    case 4: return launch_pf2<4, false, 128>(tw, tb, p, stream);
    case 5: return launch_pf2<5, false, 128>(tw, tb, p, stream);
    case 6: return launch_pf2<6, false, 128>(tw, tb, p, stream);
    case 7: return launch_pf2<7, false, 128>(tw, tb, p, stream);
    default: return launch_pf2<8, false, 128>(tw, tb, p, stream);
  }
}

}  // namespace apt
