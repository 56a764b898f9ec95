// gemm_tc.cu — APT W_p x A_q GEMM on the 5th-generation tensor cores (tcgen05, kind::i8).
//
//   D[128 weight rows x BN tokens] (s32, TMEM) += A[128 x K] (u8 digits, TMEM) . B[BN x K]^T (u8, SMEM)
//
// Per CTA: 384 threads = 12 warps, one 128 x BN output tile (BN = 16 / 64 / 128 / 256):
//   warp 0      producer (one thread): the weight planes of the CTA's K range — tile-major planes
//               (APT_PACK_TILED) with cp.async.bulk runs, canonical planes with one 3-D TMA box per
//               chunk ({words, 128 rows, wbits planes}: the paper's concatenated "unified matrix",
//               §4.1 Step 3, moved with one command) — into a ring of weight slots, the first
//               ring's worth before griddepcontrol.wait; then the token digits (2-D 128B-swizzled TMA
//               boxes of the activation digit view): the whole K range at once for BN = 16, a
//               `stages`-deep ring otherwise.
//   warp 1      MMA issuer (one thread): 4 x tcgen05.mma.cta_group::1.kind::i8 (M=128, N=BN, K=32)
//               per 128-element K step, A from the TMEM ring, B from a shared-memory descriptor;
//               tcgen05.commit frees the ring slots and finally signals the accumulator.
//   warps 2-3   TMEM allocation; epilogue operands (weight row sums / scales before the wait, token
//               row sums / scales after).
//   warps 4-11  converters (two per TMEM sub-partition, alternating K steps), then the epilogue.
//               Thread = weight row (= TMEM lane).  Per K step each thread reads its row's wbits x 16 B
//               of planes, rebuilds the 128 u8 digits with rebuild8() (the shift half of the shift-add
//               recovery) and writes them to the TMEM A ring with tcgen05.st — the planes never
//               leave the SM in any other form (recovery-oriented scheduling, §4.2).  After
//               the last MMA they load the accumulator (tcgen05.ld) and apply the rank-1 correction +
//               scale (common.cuh), or push split-K partials to the owning cluster rank over DSMEM.
//
// Token digits come from the activation digit view written by the pack kernel (apt_packed.digits),
// or from expand_tokens_kernel into the workspace, in the same within-word K order rebuild8() uses,
// so both operands agree on K.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"
#include "tc_ptx.cuh"

namespace apt {

constexpr int kTcBM = 128;       // weight rows per tile (MMA M)
constexpr int kTcBK = 128;       // K elements per pipeline step
// TMEM A ring depth (32 columns each); decode tiles (BN = 16) fit up to 7 next to the accumulator in
// 256 columns, so more weight steps are converted ahead of the token tile's arrival
#ifndef APT_DEC_NACC
#define APT_DEC_NACC 1
#endif
#ifndef APT_DEC_ASTAGES
#define APT_DEC_ASTAGES 4
#endif
#ifdef APT_TC_TRACE
// per-stage clock64 timeline of CTA (APT_TC_TRACE_CTA, 0) for profiling builds only
__device__ long long g_tc_trace[8][512];
#define TRACE(slot, ks) do { if (blockIdx.x == APT_TC_TRACE_CTA && blockIdx.y == 0 && blockIdx.z == 0 && (ks) < 512) g_tc_trace[slot][(ks)] = clock64(); } while (0)
#else
#define TRACE(slot, ks) do { } while (0)
#endif
#ifdef APT_TC_GTRACE
// grid-wide globaltimer timeline: [cta][phase], phases 0 entry 1 setup 2 first W 3 tokens 4 acc_full
// 5 split-K push start 6 exit 7 smid 8 prefetch issued 9 partials received (profiling builds only)
__device__ unsigned long long g_tc_gtrace[8192][16];
__device__ unsigned int g_tc_gtrace_next;  // next free row (reset by apt_debug_tc_gtrace_reset)
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// recorded in shared memory (a global store before a release fence would be waited for) and
// copied out once at the end
#define GTRACE(ph) do { s_gt[ph] = (ph) == 7 ? (unsigned long long)smid_u32() : gtimer_ns(); } while (0)
// rows are taken in exit order from a global counter, so consecutive launches land in distinct rows;
// column 13 holds the CTA's linear index, 14 the grid size
#define GTRACE_DUMP() do { const unsigned c_ = atomicAdd(&g_tc_gtrace_next, 1u); \
  s_gt[13] = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
  s_gt[14] = gridDim.x * gridDim.y * gridDim.z; \
  if (c_ < 8192) for (int i_ = 0; i_ < 16; ++i_) g_tc_gtrace[c_][i_] = s_gt[i_]; } while (0)
__device__ __forceinline__ uint32_t smid_u32() { uint32_t r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#else
#define GTRACE(ph) do { } while (0)
#define GTRACE_DUMP() do { } while (0)
#endif

// ------------------------------------------------------------------------------------ pre-pass
// Activation planes [abits][M][k_words] -> u8 digits [M][Kpad] in rebuild8() order (used when the
// packed activation carries no digit view).
__global__ void __launch_bounds__(256) expand_tokens_kernel(const uint32_t* __restrict__ ap, int64_t a_pstride,
                                                            int32_t M, int32_t k_words, int32_t abits,
                                                            uint8_t* __restrict__ ws) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)M * k_words) return;
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = i < abits ? __ldg(ap + (int64_t)i * a_pstride + idx) : 0u;
  uint32_t d[8];
  rebuild8_rt(w, abits, d);
  uint4* dst = reinterpret_cast<uint4*>(ws + idx * 32);
  dst[0] = make_uint4(d[0], d[1], d[2], d[3]);
  dst[1] = make_uint4(d[4], d[5], d[6], d[7]);
}

cudaError_t launch_expand_tokens(const uint32_t* ap, int64_t a_pstride, int M, int k_words, int abits, uint8_t* out,
                                 cudaStream_t stream) {
  const int64_t total = (int64_t)M * k_words;
  return launch_pdl(expand_tokens_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, stream, dim3(1, 1, 1),
                    ap, a_pstride, M, k_words, abits, out);
}

// Activation planes [abits][M][k_words] -> signed e2m1 nibbles [M][Kpad / 2] (rebuild_e2m1 order, 16
// bytes per 32-element word): the token operand of the kind::mxf4 path (abits <= 3).
__global__ void __launch_bounds__(256) expand_tokens_mx_kernel(const uint32_t* __restrict__ ap, int64_t a_pstride,
                                                               int32_t M, int32_t k_words, int32_t abits,
                                                               uint8_t* __restrict__ ws) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)M * k_words) return;
  uint32_t w[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) w[i] = i < abits ? __ldg(ap + (int64_t)i * a_pstride + idx) : 0u;
  uint32_t g[4];
  if (abits == 1) rebuild_e2m1<1>(w, g);
  else if (abits == 2) rebuild_e2m1<2>(w, g);
  else rebuild_e2m1<3>(w, g);
  *reinterpret_cast<uint4*>(ws + idx * 16) = make_uint4(g[0], g[1], g[2], g[3]);
}

cudaError_t launch_expand_tokens_mx(const uint32_t* ap, int64_t a_pstride, int M, int k_words, int abits, uint8_t* out,
                                    cudaStream_t stream) {
  const int64_t total = (int64_t)M * k_words;
  return launch_pdl(expand_tokens_mx_kernel, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, stream, dim3(1, 1, 1),
                    ap, a_pstride, M, k_words, abits, out);
}

// ------------------------------------------------------------------------------------ main kernel
template <int WB, int BN, int STAGES>
struct TcSmem {
  // weight planes move in chunks of CW words (CW*32 K elements) per row and plane (32-byte TMA rows
  // for WB <= 4); decode-sized tiles keep more chunks in flight (HBM latency x bandwidth)
  static constexpr int kCW = 8;
  static constexpr int kKpc = kCW / 4;                  // 128-element K steps per weight chunk
  // BN == 16 (decode): the CTA's whole token slab (<= kBAllSteps K steps) is loaded once up front,
  // so the TMA queue in steady state carries only the weight stream; the rest of ~113 KB (two
  // CTAs per SM) goes to weight chunks in flight
  static constexpr bool kBAll = BN == 16;
  static constexpr int kBAllSteps = 16;
  static constexpr int kWSlots = kBAll ? ((65536 / (WB * kTcBM * 8 * 4)) > 8 ? 8 : (65536 / (WB * kTcBM * 8 * 4)) < 2 ? 2 : (65536 / (WB * kTcBM * 8 * 4)))
                                       : BN <= 64 ? (WB <= 4 ? 6 : 3) : 2;
  static constexpr int kBBytes = BN * kTcBK;            // token digits per K step
  static constexpr int kWBytes = WB * kTcBM * kCW * 4;  // weight planes per chunk
  static constexpr int kBOff = 0;
  static constexpr int kWOff = (kBAll ? kBAllSteps : STAGES) * kBBytes;
  static constexpr int kRbOff = kWOff + kWSlots * kWBytes;       // split-K receive buffer: [S][128][cpr], cpr = ceil(BN / S), so S * cpr <= BN + S - 1 <= BN + 7
  static constexpr int kEpOff = kRbOff + (BN <= 64 ? kTcBM * (BN + 8) * 4 : 0);  // rw[128] ws[128] ra[BN] as[BN]
  static constexpr int kBarOff = kEpOff + (2 * kTcBM + 2 * BN) * 4;
  static constexpr int kAStages = BN == 16 ? APT_DEC_ASTAGES : 4;
  static constexpr int kNumBars = 2 * STAGES + 2 * kWSlots + 2 * kAStages + 4;
  static constexpr int kTotal = kBarOff + kNumBars * 8 + 16 + 1024;  // + tmem slot + alignment slack
};

__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(mask)
      : "memory");
}
// CN = CTAs of a cluster along the weight-row dimension sharing one token tile: each loads BN/CN
// token rows and multicasts them to all CN, so the token tile crosses L2 -> SM once per cluster.
// gridDim.z = S > 1 (with CN = 1): the K steps are split over a (1, 1, S) cluster and the S partial
// accumulator tiles are reduced through distributed shared memory (decode-sized token counts).
// MX: the kind::mxf4 variant (wbits, abits <= 3; S == 1, BN >= 128): one MMA step = one weight chunk
// = 256 K elements (both 2 KB halves of a tile-major slab), weights rebuilt as signed e2m1 nibbles
// (rebuild_e2m1) into the same 32 TMEM columns per step, tokens as the e2m1 view (128 bytes per row and
// step), 4 x tcgen05.mma kind::mxf4 (K = 64) per step into an f32 accumulator that holds the exact
// signed product (every partial sum is an integer below 2^24; reading R-MX).
template <int WB, int BN, int STAGES, int CN, bool MX>
__global__ void __launch_bounds__(384, (BN <= 128 && WB <= 4) ? 2 : 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tm_w,
                                                         const __grid_constant__ CUtensorMap tm_b, TcArgs p) {
  static_assert(!MX || (WB <= 3 && BN >= 128), "kind::mxf4 path: wbits <= 3, token tiles of 128 / 256");
  using L = TcSmem<WB, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
#ifdef APT_TC_GTRACE
  __shared__ unsigned long long s_gt[16];  // phases a launch does not reach hold garbage
#endif
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sB = base + L::kBOff;
  const uint32_t sW = base + L::kWOff;
  const uint32_t bars = base + L::kBarOff;
  int32_t* rbuf = reinterpret_cast<int32_t*>(gbase + L::kRbOff);
  int32_t* ep_rw = reinterpret_cast<int32_t*>(gbase + L::kEpOff);
  float* ep_ws = reinterpret_cast<float*>(ep_rw + kTcBM);
  int32_t* ep_ra = reinterpret_cast<int32_t*>(ep_ws + kTcBM);
  float* ep_as = reinterpret_cast<float*>(ep_ra + BN);
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (STAGES + s); };
  auto wfull = [&](int c) { return bars + 8u * (2 * STAGES + c); };
  auto wempty = [&](int c) { return bars + 8u * (2 * STAGES + L::kWSlots + c); };
  auto a_full = [&](int a) { return bars + 8u * (2 * STAGES + 2 * L::kWSlots + a); };
  auto a_empty = [&](int a) { return bars + 8u * (2 * STAGES + 2 * L::kWSlots + L::kAStages + a); };
  const uint32_t acc_full = bars + 8u * (2 * STAGES + 2 * L::kWSlots + 2 * L::kAStages);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + L::kBarOff + L::kNumBars * 8);
  // decode tiles (BN = 16): the four 32-element MMAs of a K step go to four independent accumulators
  // (summed in the epilogue), so consecutive MMAs carry no accumulator dependency and pipeline in the
  // tensor core instead of serialising on the MMA latency
  constexpr int kNAcc = BN == 16 ? APT_DEC_NACC : 1;
  constexpr uint32_t kSfCols = MX ? 32 : 0;  // unit scale factors (mxf4): 16 columns for A, 16 for B
  constexpr uint32_t kTmemCols = (BN * kNAcc + 32 * L::kAStages + kSfCols) <= 256 ? 256 : 512;
  constexpr uint32_t kAcol0 = BN * kNAcc;  // A ring after the accumulator columns
  constexpr uint32_t kScol0 = kAcol0 + 32 * L::kAStages;
  constexpr int kRowsPerCta = BN / CN;
  constexpr uint16_t kMask = (uint16_t)((1u << CN) - 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kTcBM;   // weight rows
  const int m0 = blockIdx.y * BN;      // tokens
  const int S = gridDim.z;             // K split (cluster along z)
  const uint32_t crank = (CN > 1 || S > 1) ? cluster_ctarank() : 0u;
  // this CTA's K steps, in whole weight chunks
  // this CTA's K steps [kb, ke): an even split at step granularity (a weight chunk is two steps
  // relative to kb; the tile-major layout keeps steps contiguous across chunk boundaries)
  const int nk = p.k_words / 4;
  const int kb = (int)(((int64_t)blockIdx.z * nk) / S);
  const int ke = (int)(((int64_t)(blockIdx.z + 1) * nk) / S);
  const int nloc = ke - kb;
  const int nms = MX ? nloc / 2 : nloc;  // MMA steps (mxf4: 256 K elements = one weight chunk each)
  pdl_launch_dependents();
  if (threadIdx.x == 0) { TRACE(6, 0); GTRACE(0); GTRACE(7); }

  // split-K over DSMEM (BN <= 64, CN == 1): rank q reduces token columns [q*cpr, q*cpr + ncols(q))
  const bool dsm = BN <= 64 && S > 1;
  const int cpr = (BN + S - 1) / S;
  auto ncols = [&](int q) { return max(0, min(cpr, BN - q * cpr)); };
  const uint32_t red_full = acc_full + 8u;
  const uint32_t wbig0 = acc_full + 16u;  // up-front weight prefetch, first chunk (one phase only)
  const uint32_t wbig = acc_full + 24u;   // up-front weight prefetch, the rest (one phase only)

  // tile-major weights (APT_PACK_TILED): a plane's K steps are contiguous 2 KB blocks in HBM, so the
  // ring is plane-major [plane][slot][2 steps x 2 KB] and a run of steps moves with one bulk copy per
  // plane (fewer, larger requests).  Canonical planes: one 3-D TMA box per chunk, chunk-major ring.
  const bool tiled = p.w_tiled != 0;
  const uint32_t* wtile = p.wp + (int64_t)(n0 >> 7) * (p.k_words >> 3) * 1024;
  auto w_run = [&](int j0, int steps, int slot, uint32_t bar) {  // steps [j0, j0 + steps) -> slot..
#pragma unroll
    for (int i = 0; i < WB; ++i)
      bulk_load(sW + (i * L::kWSlots + slot) * 4096, wtile + (int64_t)i * p.w_pstride + (int64_t)(kb + j0) * 512,
                (uint32_t)steps * 2048, bar);
  };
  auto issue_w = [&](int c) {  // weight chunk c (local steps 2c, 2c + 1)
    const int slot = c % L::kWSlots;
    mbar_wait(wempty(slot), ((c / L::kWSlots) & 1) ^ 1);
    // the converters' generic-proxy reads of this slot (released through wempty) before the async-proxy
    // (bulk copy / TMA) overwrite: a proxy fence makes the write-after-read order explicit
    fence_proxy_async();
    if (tiled) {
      const int steps = min(2, nloc - 2 * c);
      mbar_expect_tx(wfull(slot), (uint32_t)(steps * 2048 * WB));
      w_run(2 * c, steps, slot, wfull(slot));
    } else {
      mbar_expect_tx(wfull(slot), L::kWBytes);
      tma_load_3d(sW + slot * L::kWBytes, &tm_w, wfull(slot), (kb + 2 * c) * 4, n0, 0);
    }
  };
  const int n_pre = min(L::kWSlots, (nloc + 1) / 2);
  const int pre_s0 = min(2, min(nloc, 2 * n_pre));  // steps in the first prefetch run
  // part: 1 = first run only, 2 = the rest only, 3 = both
  auto issue_pre = [&](int part) {
    if (tiled) {
      // the first ring's worth of steps in two runs per plane: chunk 0 (conversion starts as soon as
      // it lands) and the rest
      const int pre = min(nloc, 2 * n_pre);
      const int s0 = pre_s0;
      if ((part & 1) && s0 > 0) {
        mbar_expect_tx(wbig0, (uint32_t)(s0 * 2048 * WB));
        w_run(0, s0, 0, wbig0);
      }
      if (!(part & 2)) return;
      if (pre > s0) {
        mbar_expect_tx(wbig, (uint32_t)((pre - s0) * 2048 * WB));
        w_run(s0, pre - s0, s0 / 2, wbig);
      }
      // these chunks complete wbig0 / wbig, not the slots' own barriers: a slot's first wfull phase
      // is its second use (chunk c + kWSlots; chunks beyond the prefetch exist only when
      // n_pre == kWSlots), see the converters' parity
    } else {
      if (part & 2)
        for (int c = 0; c < n_pre; ++c) issue_w(c);
    }
  };
  // decode tiles: only the first weight run goes out before griddepcontrol.wait; the token slab is
  // requested right after the wait, ahead of the rest of the weight prefetch (else it queues behind
  // ~64 KB of weight copies per CTA and the MMA idles ~0.6 us)
#ifdef APT_DEC_TOK_EARLY
  constexpr bool kTokEarly = L::kBAll && CN == 1;
#else
  constexpr bool kTokEarly = false;
#endif

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), CN);      // every cluster CTA's MMA commit (multicast when CN > 1)
    }
    for (int c = 0; c < L::kWSlots; ++c) {
      mbar_init(wfull(c), 1);
      mbar_init(wempty(c), MX ? 4 : 8);  // the converter warps reading the chunk (one step each; mxf4: one parity)
    }
    for (int a = 0; a < L::kAStages; ++a) {
      mbar_init(a_full(a), 4);
      mbar_init(a_empty(a), 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(red_full, 1);
    mbar_init(wbig0, 1);
    mbar_init(wbig, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the partial tiles this rank will receive (st.async complete_tx from every rank, itself included)
    if (dsm) mbar_expect_tx(red_full, (uint32_t)(S * kTcBM * ncols((int)crank) * 4));
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_w) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
    // weights never depend on the previous kernel (programmatic dependent launch) and need nothing
    // but this thread's barriers: the first ring's worth of chunks is requested before the rest of
    // the setup (TMEM allocation, CTA / cluster barriers)
#ifndef APT_TC_LATE_W
    if (CN == 1) issue_pre(kTokEarly && tiled ? 1 : 3);
#endif
    GTRACE(8);
  }
  if (warp == 4 && lane == 0) GTRACE(12);
  if (warp == 2) {
    if (lane == 0) GTRACE(10);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    if (lane == 0) GTRACE(11);
  }
  tc_fence_before();
  if (CN > 1) {
    cluster_sync_all();  // multicast writes into peers from the first token tile on
  } else {
    __syncthreads();
    // split-K peers are first touched at the reduction: arrive now, wait right before it.  Relaxed:
    // the barrier inits are already released by fence.mbarrier_init, and a release arrive would wait
    // for this thread's outstanding weight bulk copies (~1-2 us)
    if (dsm) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  }
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(tmem_slot);
  if (threadIdx.x == 0) { TRACE(6, 1); GTRACE(1); }

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
#ifndef APT_TC_LATE_W
      if (CN > 1)
#endif
        issue_pre(3);
      pdl_wait();
      GTRACE(15);
      if constexpr (L::kBAll) {
        // the whole token slab of this CTA's K range, one barrier.  (Requesting it from another warp
        // ahead of the weight prefetch measured 5% slower in back-to-back launches.)
        mbar_expect_tx(full(0), (uint32_t)(nloc * L::kBBytes));
        for (int j = 0; j < nloc; ++j) tma_load_2d(sB + j * L::kBBytes, &tm_b, full(0), (kb + j) * kTcBK, m0);
        if (kTokEarly && tiled) issue_pre(2);
      }
      if constexpr (MX) {
        for (int j = 0; j < nms; ++j) {
          if (j >= n_pre) issue_w(j);  // weight chunk j = MMA step j
          const int s = j % STAGES;
          mbar_wait(empty(s), ((j / STAGES) & 1) ^ 1);
          mbar_expect_tx(full(s), L::kBBytes);
          tma_load_2d(sB + s * L::kBBytes, &tm_b, full(s), (kb / 2 + j) * 128, m0);  // 128 bytes = 256 K
        }
      }
      for (int j = 0; j < (MX ? 0 : nloc); ++j) {
        const int ks = kb + j;
        if (j % 2 == 0 && j / 2 >= n_pre) {  // next weight chunk
          issue_w(j / 2);
        }
        if constexpr (L::kBAll) continue;
        const int s = j % STAGES;
        const uint32_t ph = (j / STAGES) & 1;
        mbar_wait(empty(s), ph ^ 1);
        TRACE(0, j);
        mbar_expect_tx(full(s), L::kBBytes);
        const uint32_t mc_rank = CN > 1 ? crank : 0u;  // cluster rank along x (multicast), not the K split
        const uint32_t dstB = sB + s * L::kBBytes + mc_rank * kRowsPerCta * kTcBK;
        if (CN > 1)
          tma_load_2d_mc(dstB, &tm_b, full(s), ks * kTcBK, m0 + (int)crank * kRowsPerCta, kMask);
        else
          tma_load_2d(dstB, &tm_b, full(s), ks * kTcBK, m0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = MX ? ((1u << 7) | (1u << 10)              // A, B = e2m1
                                        | ((uint32_t)(BN >> 3) << 17)     // N
                                        | (1u << 23)                      // scale factors UE8M0
                                        | ((uint32_t)(kTcBM >> 4) << 24))  // M ; K-major
                                     : ((2u << 4)                         // D = s32
                                        | ((uint32_t)(BN >> 3) << 17)     // N
                                        | ((uint32_t)(kTcBM >> 4) << 24));  // M ; A, B = u8, K-major
      for (int j = 0; j < nms; ++j) {
        const int s = L::kBAll ? j : j % STAGES;
        const uint32_t ph = (j / STAGES) & 1;
        const int a = j % L::kAStages;
        const uint32_t pa = (j / L::kAStages) & 1;
        if (!L::kBAll || j == 0) mbar_wait(full(L::kBAll ? 0 : s), L::kBAll ? 0u : ph);
        TRACE(1, j);
        if (j == 0) GTRACE(3);
        mbar_wait(a_full(a), pa);
        TRACE(2, j);
        tc_fence_after();
        const uint64_t bdesc = umma_desc_sw128(sB + s * L::kBBytes);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // advance 32 bytes (32 u8 / 64 e2m1) inside the 128-byte swizzle atom: +2 in the (addr >> 4) field
          if constexpr (MX)
            tc_mma_mxf4(tmem, tmem + kAcol0 + 32 * a + 8 * kk, bdesc + (uint64_t)(2 * kk), idesc, (j | kk) != 0,
                        tmem + kScol0, tmem + kScol0 + 16);
          else
            tc_mma_i8(tmem + (uint32_t)((kk % kNAcc) * BN), tmem + kAcol0 + 32 * a + 8 * kk, bdesc + (uint64_t)(2 * kk),
                      idesc, (kNAcc > 1 ? (j | (kk / kNAcc)) : (j | kk)) != 0);
        }
        if (!L::kBAll) {
          if (CN > 1) tc_commit_mc(empty(s), kMask); else tc_commit(empty(s));
        }
        tc_commit(a_empty(a));
      }
      tc_commit(acc_full);
    }
  } else if (warp < 4) {
    // ------------------------------------------------------------ epilogue operands (warps 2, 3)
    for (int i = threadIdx.x - 64; i < kTcBM; i += 64) {  // weight side: immutable
      const int n = min(n0 + i, p.e.N - 1);
      ep_rw[i] = __ldg(p.e.w_rowsum + n);
      ep_ws[i] = p.e.kind == 2 ? __ldg(p.e.w_scale + n) : 0.f;
    }
    pdl_wait();  // token side: written by the previous kernel (the activation pack)
    for (int i = threadIdx.x - 64; i < BN; i += 64) {
      const int m = min(m0 + i, p.e.M - 1);
      ep_ra[i] = __ldg(p.e.a_rowsum + m);
      ep_as[i] = (p.e.kind == 2 && p.e.a_scale) ? __ldg(p.e.a_scale + m) : 1.f;
    }
    asm volatile("bar.arrive 1, 320;" ::: "memory");
  } else {
    // ------------------------------------------------------------ converters (warps 4..11)
    // two warps per TMEM sub-partition: parity `par` converts the K steps j with j % 2 == par, so
    // one warp's shared-memory / rebuild / tcgen05.st latency overlaps the other's
    const int cw = warp - 4, sub = cw & 3, par = cw >> 2;
    const int r = sub * 32 + lane;       // row within the tile (= TMEM lane)
    const uint32_t lane_off = (uint32_t)(sub * 32) << 16;
#ifdef APT_CONV_PIPE
    int pend_a = -1;  // A stage whose tcgen05.st is still in flight
#endif
    if constexpr (MX) {
      // unit UE8M0 scale factors (2^0) for every row / column the MMAs read: parity 0 of each
      // sub-partition fills its 32 lanes of the 32 scale columns before its first a_full arrive
      if (par == 0) {
        uint32_t one[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) one[i] = 0x7F7F7F7Fu;
        tmem_st32<32>(tmem + lane_off + kScol0, one);
      }
    }
    for (int j = par; j < nms; j += 2) {
      const int c = MX ? j : j / L::kKpc, q = MX ? 0 : j % L::kKpc;  // kKpc == 2: each parity reads one step per chunk
      if (tiled && c < n_pre) mbar_wait(2 * c < pre_s0 ? wbig0 : wbig, 0);
      else mbar_wait(wfull(c % L::kWSlots), ((c / L::kWSlots) - (tiled ? 1 : 0)) & 1);
      if (lane == 0 && (cw & 3) == 0) TRACE(3, j);
      if (lane == 0 && cw == 0 && j == 0) GTRACE(2);
      constexpr int kH = MX ? 2 : 1;  // 16-byte pieces per plane and row (mxf4 steps read both halves)
      uint4 v[kH][WB];
      const uint8_t* wsm = gbase + L::kWOff;
#pragma unroll
      for (int h = 0; h < kH; ++h)
#pragma unroll
        for (int i = 0; i < WB; ++i) {
          const int off = tiled ? (i * L::kWSlots + c % L::kWSlots) * 4096 : (c % L::kWSlots) * L::kWBytes + i * 4096;
          // tile-major: [q][row][4 words] (lanes read consecutive 16 B); canonical TMA box: [row][8 words]
          const int qq = MX ? h : q;
          v[h][i] = *reinterpret_cast<const uint4*>(wsm + off + (p.w_tiled ? qq * 2048 + r * 16 : (r * L::kCW + 4 * qq) * 4));
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(wempty(c % L::kWSlots));
      uint32_t d[32];
      if constexpr (MX) {
        // 8 words x 16 bytes of signed e2m1 nibbles (word wi -> TMEM columns 4 wi .. 4 wi + 3)
#pragma unroll
        for (int wi = 0; wi < 8; ++wi) {
          uint32_t w[3] = {0u, 0u, 0u}, g[4];
#pragma unroll
          for (int i = 0; i < WB; ++i) {
            const uint4& t = v[wi >> 2][i];
            const int jj = wi & 3;
            w[i] = jj == 0 ? t.x : jj == 1 ? t.y : jj == 2 ? t.z : t.w;
          }
          if constexpr (MX) rebuild_e2m1<(WB <= 3 ? WB : 3)>(w, g);
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) d[4 * wi + cc] = g[cc];
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t w[WB], o[8];
#pragma unroll
          for (int i = 0; i < WB; ++i) w[i] = jj == 0 ? v[0][i].x : jj == 1 ? v[0][i].y : jj == 2 ? v[0][i].z : v[0][i].w;
          rebuild8<WB>(w, o);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) d[8 * jj + cc] = o[cc];
        }
      }
      const int a = j % L::kAStages;
      const uint32_t pa = (j / L::kAStages) & 1;
      if (lane == 0 && (cw & 3) == 0) TRACE(7, j);
#ifdef APT_CONV_PIPE
      // the previous step's TMEM store completed while this step was rebuilt: publish it now
      if (pend_a >= 0) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(a_full(pend_a));
      }
      mbar_wait(a_empty(a), pa ^ 1);
      tc_fence_after();
      tmem_st32<32>(tmem + lane_off + kAcol0 + 32 * a, d);
      pend_a = a;
#else
      mbar_wait(a_empty(a), pa ^ 1);
      tc_fence_after();
      tmem_st32<32>(tmem + lane_off + kAcol0 + 32 * a, d);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full(a));
#endif
      if (lane == 0 && (cw & 3) == 0) TRACE(4, j);
    }
#ifdef APT_CONV_PIPE
    if (pend_a >= 0) {
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full(pend_a));
    }
#endif
    // ------------------------------------------------------------ epilogue
    // warp (sub, par) owns rows 32*sub.. and the token columns [par*BN/2, (par+1)*BN/2)
    asm volatile("bar.sync 1, 320;" ::: "memory");   // epilogue operands are in shared memory
    mbar_wait(acc_full, 0);
    if (lane == 0 && cw == 0) { TRACE(5, 0); GTRACE(4); }
    tc_fence_after();
    constexpr int kHalf = BN / 2;
    constexpr int kChunk = kHalf < 32 ? kHalf : 32;
    auto load_acc = [&](int c0, uint32_t (&acc)[kChunk]) {
      tmem_ld<kChunk>(tmem + lane_off + c0, acc);
#pragma unroll
      for (int q = 1; q < kNAcc; ++q) {
        uint32_t t[kChunk];
        tmem_ld<kChunk>(tmem + lane_off + (uint32_t)(q * BN) + c0, t);
#pragma unroll
        for (int jj = 0; jj < kChunk; ++jj) acc[jj] += t[jj];
      }
    };
    const int n = n0 + r;
    const int32_t rw = ep_rw[r];
    const float wsc = ep_ws[r];
    if (S == 1) {
#pragma unroll 1
      for (int c0 = par * kHalf; c0 < (par + 1) * kHalf; c0 += kChunk) {
        uint32_t acc[kChunk];
        load_acc(c0, acc);
        if constexpr (MX) {  // f32 accumulator holding an exact integer -> the signed product
#pragma unroll
          for (int jj = 0; jj < kChunk; ++jj) acc[jj] = (uint32_t)__float2int_rn(__uint_as_float(acc[jj]));
        }
        if (n < p.e.N) {
          if (p.e.kind == 2) {
            // fp16 (the common case): the rank-1 terms of the row hoisted, one fp32 expression per
            // element, then either 2-byte stores (row layout: the warp's lanes are consecutive n, so
            // each store instruction is coalesced) or 16-byte stores of 8 tokens (column layout)
            const uint32_t cn = (uint32_t)p.e.h_a * (uint32_t)rw + (uint32_t)p.e.kpad * (uint32_t)p.e.h_a * (uint32_t)p.e.h_w;
            const int mb = m0 + c0;
            uint32_t hv[kChunk / 2];
#pragma unroll
            for (int jj = 0; jj < kChunk; jj += 2) {
              float v2[2];
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) {
                const uint32_t y = acc[jj + e2] - (uint32_t)p.e.h_w * (uint32_t)ep_ra[c0 + jj + e2] - cn;
                v2[e2] = ((float)(int32_t)y * wsc) * ep_as[c0 + jj + e2];
              }
              hv[jj / 2] = pack_f16x2(v2[0], v2[1]);
            }
            unsigned short* outh = reinterpret_cast<unsigned short*>(p.e.out);
            if (p.e.layout == 0) {
              unsigned short* q = outh + (int64_t)mb * p.e.ldo + n;
#pragma unroll
              for (int jj = 0; jj < kChunk; ++jj)
                if (mb + jj < p.e.M) q[(int64_t)jj * p.e.ldo] = (unsigned short)(hv[jj / 2] >> (16 * (jj & 1)));
            } else {
              unsigned short* q = outh + (int64_t)n * p.e.ldo + mb;
              if (mb + kChunk <= p.e.M && ((reinterpret_cast<uintptr_t>(q) & 15u) == 0)) {
#pragma unroll
                for (int jj = 0; jj < kChunk; jj += 8)
                  *reinterpret_cast<uint4*>(q + jj) = make_uint4(hv[jj / 2], hv[jj / 2 + 1], hv[jj / 2 + 2], hv[jj / 2 + 3]);
              } else {
#pragma unroll
                for (int jj = 0; jj < kChunk; ++jj)
                  if (mb + jj < p.e.M) q[jj] = (unsigned short)(hv[jj / 2] >> (16 * (jj & 1)));
              }
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < kChunk; ++jj) {
              const int m = m0 + c0 + jj;
              if (m < p.e.M) epilogue_store_v(p.e, m, n, acc[jj], ep_ra[c0 + jj], rw, wsc, ep_as[c0 + jj]);
            }
          }
        }
      }
    } else if constexpr (BN <= 64) {
      // ---------------------------------------------------------- split-K: push partials over DSMEM
      // token column col goes to rank col / cpr, slot col % cpr of that rank's rbuf[src = crank][r][.],
      // as st.async stores that count down the receiver's red_full barrier
      __syncwarp();
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' barriers initialised
      if (lane == 0 && cw == 0) GTRACE(5);
      const uint32_t rb_local = smem_u32(rbuf) + (uint32_t)(((int)crank * kTcBM + r) * cpr * 4);
      const int vec = (cpr % 4 == 0) ? 4 : (cpr % 2 == 0) ? 2 : 1;
#pragma unroll 1
      for (int c0 = par * kHalf; c0 < (par + 1) * kHalf; c0 += kChunk) {
        uint32_t acc[kChunk];
        load_acc(c0, acc);
        if (nloc == 0) {  // an empty K range (more splits than weight chunks) contributes zero
#pragma unroll
          for (int jj = 0; jj < kChunk; ++jj) acc[jj] = 0u;
        }
#pragma unroll
        for (int jj = 0; jj < kChunk; jj += 4) {
#pragma unroll
          for (int h = 0; h < 4; h += vec) {
            const int col = c0 + jj + h;
            const int q = col / cpr;
            uint32_t raddr, rbar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(rb_local + (uint32_t)((col - q * cpr) * 4)), "r"(q));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(red_full), "r"(q));
            if (vec == 4)
              asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                           ::"r"(raddr), "r"(acc[jj + h]), "r"(acc[jj + h + 1]), "r"(acc[jj + h + 2]), "r"(acc[jj + h + 3]),
                           "r"(rbar) : "memory");
            else if (vec == 2)
              asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];"
                           ::"r"(raddr), "r"(acc[jj + h]), "r"(acc[jj + h + 1]), "r"(rbar) : "memory");
            else
              asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                           ::"r"(raddr), "r"(acc[jj + h]), "r"(rbar) : "memory");
          }
        }
      }
      __syncwarp();
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // exit guard (see below)
      // this rank's columns: the sum of the S partials, then the epilogue
      mbar_wait_cluster(red_full, 0);
      if (lane == 0 && cw == 0) GTRACE(9);
      const int nc = ncols((int)crank);
      for (int sl = par; sl < nc; sl += 2) {
        const int col = (int)crank * cpr + sl;
        const int m = m0 + col;
        if (m < p.e.M && n < p.e.N) {
          uint32_t U = 0;
          for (int src = 0; src < S; ++src) U += (uint32_t)rbuf[(src * kTcBM + r) * cpr + sl];
          epilogue_store_v(p.e, m, n, U, ep_ra[col], rw, wsc, ep_as[col]);
        }
      }
    }
  }
  if (dsm && warp < 4) {
    // the other warps take part in both cluster barrier phases
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  if (warp == 4 && lane == 0) TRACE(5, 1);
  if (threadIdx.x == 0) TRACE(5, 2);
  tc_fence_before();
  __syncwarp();  // reconverge the role-divergent warps before the .aligned barriers
  // no CTA may leave while cluster peers can still multicast / st.async into it or signal its barriers
  if (CN > 1) cluster_sync_all();
  else if (dsm) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (threadIdx.x == 0) { GTRACE(6); GTRACE_DUMP(); }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

// ------------------------------------------------------------------------------------ host side
PFN_encodeTiled_t tensor_map_encoder() {
  // resolved once (thread-safe static initialization)
  static const PFN_encodeTiled_t fn = []() -> PFN_encodeTiled_t {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_encodeTiled_t>(ptr);
    cudaGetLastError();
    return nullptr;
  }();
  return fn;
}

bool make_plane_map(CUtensorMap* map, const uint32_t* planes, int k_words, int rows, int bits, int box_words,
                    int box_rows) {
  PFN_encodeTiled_t enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)k_words, (cuuint64_t)rows, (cuuint64_t)bits};
  cuuint64_t strides[2] = {(cuuint64_t)k_words * 4, (cuuint64_t)k_words * 4 * (cuuint64_t)rows};
  cuuint32_t box[3] = {(cuuint32_t)box_words, (cuuint32_t)box_rows, (cuuint32_t)bits};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(planes), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__host__ __device__ constexpr int tc_clamp(int v, int lo, int hi) { return v < lo ? lo : v > hi ? hi : v; }

__host__ __device__ constexpr int tc_stages_ct(int wbits, int bn) {
  // token-tile ring as deep as shared memory allows next to the weight-chunk ring: ~108 KB per CTA
  // at BN <= 128 (two CTAs per SM), ~216 KB at 256
  return tc_clamp(((bn <= 128 ? 108 : 216) * 1024 -
                   (bn <= 64 ? (wbits <= 4 ? 6 : 3) : 2) * wbits * kTcBM * 8 * 4 -
                   (bn <= 64 ? kTcBM * (bn + 8) * 4 : 0) - 4096) / (bn * kTcBK),
                  2, 8);
}

int tc_stages(int wbits, int bn) { return tc_stages_ct(wbits, bn); }

size_t tc_workspace_bytes(int M, int k_words) { return (size_t)M * (size_t)k_words * 32u; }

template <int WB, int BN, int ST, int CN, bool MX = false>
static cudaError_t launch_tc4(const CUtensorMap& tw, const CUtensorMap& tb, const TcArgs& p, int split,
                              cudaStream_t stream) {
  using L = TcSmem<WB, BN, ST>;
  static_assert(L::kTotal <= 227 * 1024, "shared memory budget");
  // the decode tiles are sized for two CTAs per SM (228 KB per SM, 1 KB reserved per CTA)
  static_assert(BN != 16 || 2 * (L::kTotal + 1024) <= 228 * 1024, "two CTAs per SM");
  auto kern = gemm_tc_kernel<WB, BN, ST, CN, MX>;
  cudaError_t err = set_smem_once<gemm_tc_kernel<WB, BN, ST, CN, MX>>(L::kTotal);
  if (err != cudaSuccess) return err;
  const int gx = ((p.e.N + kTcBM - 1) / kTcBM + CN - 1) / CN * CN;
  return launch_pdl(kern, dim3(gx, (p.e.M + BN - 1) / BN, split), dim3(384), L::kTotal, stream, dim3(CN, 1, split),
                    tw, tb, p);
}

template <int WB, int BN>
static cudaError_t launch_tc2(const CUtensorMap& tw, const CUtensorMap& tb, const TcArgs& p, int cn, int split,
                              cudaStream_t stream) {
  constexpr int ST = tc_stages_ct(WB, BN);
  if constexpr (BN < 128) {
    return launch_tc4<WB, BN, ST, 1>(tw, tb, p, split, stream);
  } else {
    switch (cn) {
      case 1: return launch_tc4<WB, BN, ST, 1>(tw, tb, p, split, stream);
      case 2: return launch_tc4<WB, BN, ST, 2>(tw, tb, p, split, stream);
      default: return launch_tc4<WB, BN, ST, 4>(tw, tb, p, split, stream);
    }
  }
}

template <int WB>
static cudaError_t launch_tc1(const CUtensorMap& tw, const CUtensorMap& tb, const TcArgs& p, int bn, int cn,
                              int split, cudaStream_t stream) {
  switch (bn) {
    case 16: return launch_tc2<WB, 16>(tw, tb, p, cn, split, stream);
    case 64: return launch_tc2<WB, 64>(tw, tb, p, cn, split, stream);
    case 256: return launch_tc2<WB, 256>(tw, tb, p, cn, split, stream);
    default: return launch_tc2<WB, 128>(tw, tb, p, cn, split, stream);
  }
}

cudaError_t launch_gemm_tc(const TcArgs& p, int wbits, int bn, int cluster_n, int split, int mx, cudaStream_t stream) {
  PFN_encodeTiled_t enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tw, tb;
  const int cw = 8;
  if (!make_plane_map(&tw, p.wp, p.k_words, p.e.N, wbits, cw, kTcBM)) return cudaErrorInvalidValue;
  {
    // token view: u8 digits [M][Kpad] (i8), or e2m1 nibbles [M][Kpad / 2] (mxf4); 128-byte boxes
    const cuuint64_t kp = (cuuint64_t)p.k_words * (mx ? 16 : 32);
    cuuint64_t dims[2] = {kp, (cuuint64_t)p.e.M};
    cuuint64_t strides[1] = {kp};
    cuuint32_t box[2] = {(cuuint32_t)kTcBK, (cuuint32_t)(bn / cluster_n)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(p.adig), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  if (mx) {  // kind::mxf4: wbits <= 3, S = 1, CN = 1, BN 128 / 256 (validated by the caller)
    switch (wbits * 1000 + bn) {
      case 1128: return launch_tc4<1, 128, tc_stages_ct(1, 128), 1, true>(tw, tb, p, 1, stream);
      case 1256: return launch_tc4<1, 256, tc_stages_ct(1, 256), 1, true>(tw, tb, p, 1, stream);
      case 2128: return launch_tc4<2, 128, tc_stages_ct(2, 128), 1, true>(tw, tb, p, 1, stream);
      case 2256: return launch_tc4<2, 256, tc_stages_ct(2, 256), 1, true>(tw, tb, p, 1, stream);
      case 3128: return launch_tc4<3, 128, tc_stages_ct(3, 128), 1, true>(tw, tb, p, 1, stream);
      case 3256: return launch_tc4<3, 256, tc_stages_ct(3, 256), 1, true>(tw, tb, p, 1, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (wbits) {
    case 1: return launch_tc1<1>(tw, tb, p, bn, cluster_n, split, stream);
    case 2: return launch_tc1<2>(tw, tb, p, bn, cluster_n, split, stream);
    case 3: return launch_tc1<3>(tw, tb, p, bn, cluster_n, split, stream);
    case 4: return launch_tc1<4>(tw, tb, p, bn, cluster_n, split, stream);
    case 5: return launch_tc1<5>(tw, tb, p, bn, cluster_n, split, stream);
    case 6: return launch_tc1<6>(tw, tb, p, bn, cluster_n, split, stream);
    case 7: return launch_tc1<7>(tw, tb, p, bn, cluster_n, split, stream);
    default: return launch_tc1<8>(tw, tb, p, bn, cluster_n, split, stream);
  }
}

}  // namespace apt

#ifdef APT_TC_GTRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_tc_gtrace_reset() {
  const unsigned z = 0;
  cudaMemcpyToSymbol(apt::g_tc_gtrace_next, &z, sizeof(z));
  return (int)cudaMemset(apt::g_tc_gtrace, 0, 0) ;
}
extern "C" __attribute__((visibility("default"))) int apt_debug_tc_gtrace(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, apt::g_tc_gtrace, sizeof(unsigned long long) * (n < 8192 * 16 ? n : 8192 * 16));
}
#endif
#ifdef APT_TC_TRACE
extern "C" __attribute__((visibility("default"))) int apt_debug_tc_trace(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, apt::g_tc_trace, sizeof(long long) * (n < 8 * 512 ? n : 8 * 512));
}
#endif
