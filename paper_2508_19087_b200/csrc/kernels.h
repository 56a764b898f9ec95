// kernels.h — launch interfaces between the C-ABI shim (apt.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace apt {

struct PackArgs {
  const int8_t* codes;
  int64_t ld;
  int32_t rows, k, k_words, enc;
  uint32_t* planes;
  int64_t plane_stride;  // rows * k_words
  int32_t* row_sum;
  int32_t* range_error;
  uint8_t* digits;       // optional [rows][Kpad] kernel-order u8 digits
  int32_t tiled;         // planes tile-major (APT_PACK_TILED)
};
cudaError_t launch_pack(const PackArgs& p, int bits, cudaStream_t stream);
// fused fp16 -> per-row symmetric quantize -> pack (x: const __half*, scale: [rows] fp32 out)
cudaError_t launch_quant_pack(const PackArgs& p, const void* x, float* scale, int bits, cudaStream_t stream);

// grouped activation packs (one word per thread, digit views): problem i owns CTAs [cta_end[i-1], cta_end[i])
constexpr int kPackGroupMax = 64;
struct PackGroupArgs {
  int32_t count;
  int32_t cta_end[kPackGroupMax];
  int32_t rows_per_cta[kPackGroupMax];
  int32_t bits[kPackGroupMax];
  const void* x[kPackGroupMax];   // fp16 rows to quantize (apt_quantize_pack semantics), or null: int8 codes
  float* scale[kPackGroupMax];    // per-row scales out (quantize)
  PackArgs p[kPackGroupMax];
};
int pack_group_rows_per_cta(const PackArgs& p);
int pack_group_threads(const PackArgs& p);
cudaError_t launch_pack_grouped(const PackGroupArgs& a, int ctas, int threads, cudaStream_t stream);

// activation planes [abits][M][k_words] -> kernel-order u8 digits [M][Kpad]
cudaError_t launch_expand_tokens(const uint32_t* ap, int64_t a_pstride, int M, int k_words, int abits,
                                 uint8_t* out, cudaStream_t stream);

}  // namespace apt

namespace apt {
struct TcArgs {
  const uint32_t* wp;      // weight planes [wbits][N][k_words] or tile-major (w_tiled)
  int64_t w_pstride;       // words per plane
  int32_t w_tiled;
  const uint8_t* adig;     // activation digits [M][Kpad], kernel K order (TMA source)
  int32_t k_words;
  EpilogueArgs e;
};
cudaError_t launch_gemm_tc(const TcArgs& p, int wbits, int bn, int cluster_n, int split, int mx, cudaStream_t stream);
// persistent tcgen05 GEMM (gemm_pf.cu): 128 x 128 tiles walked by one CTA per SM, double-buffered
// accumulator; mx = kind::mxf4 (tokens = the e2m1 view)
cudaError_t launch_gemm_pf(const TcArgs& p, int wbits, int mx, int bn, cudaStream_t stream);
// activation planes -> signed e2m1 token view [M][Kpad / 2] for the kind::mxf4 path (abits <= 3)
cudaError_t launch_expand_tokens_mx(const uint32_t* ap, int64_t a_pstride, int M, int k_words, int abits, uint8_t* out,
                                    cudaStream_t stream);
int tc_stages(int wbits, int bn);
size_t tc_workspace_bytes(int M, int k_words);
}  // namespace apt

namespace apt {
struct GemvArgs {
  const uint32_t* wp;      // weight planes (row or tile-major layout)
  int64_t w_pstride;       // words per plane
  int32_t w_tiled;
  const uint8_t* adig;     // activation digits [M][Kpad], kernel K order
  int32_t k_words;
  EpilogueArgs e;
};
// M <= 4 tokens: SIMT dp4a GEMV over rebuilt weight digits (gemv.cu)
cudaError_t launch_gemv(const GemvArgs& p, int wbits, int warps, cudaStream_t stream);  // warps: 8 or 16
// M <= 16: mma.sync m16n8k32 u8 skinny GEMM fed from registers (gemm_skinny.cu); bn 8 or 16, warps 4/8/16
cudaError_t launch_gemm_skinny(const GemvArgs& p, int wbits, int bn, int warps, cudaStream_t stream);

// M <= 16: mma.sync m16n8k32 u8 with the weights as the streamed B operand and the tokens resident in
// registers (gemm_dec.cu); 32 weight rows per CTA of `warps` (4 / 8) warps splitting K, split = CTAs
// along K (> 1 needs the partials + tickets workspace, tickets zero before the first call and left zero)
struct DecArgs {
  const uint32_t* wp;      // weight planes (row or tile-major layout)
  int64_t w_pstride;       // words per plane
  int32_t w_tiled;
  const uint8_t* adig;     // activation digits [M][Kpad], kernel K order
  int32_t k_words;
  EpilogueArgs e;
  int32_t* partials;       // [tiles][split][16][32] int32 (split > 1)
  uint32_t* counters;      // [tiles] tickets (split > 1)
};
cudaError_t launch_gemm_dec(const DecArgs& p, int wbits, int warps, int split, cudaStream_t stream);
size_t dec_workspace_bytes(int N, int split);
int dec_blocks_per_cta(int k_words, int split);
}  // namespace apt

namespace apt {
// fp16 output with zero points from the exact int32 Y (epilogue_zp.cu)
struct ZpArgs {
  const int32_t* y;         // [M][N] row-major, signed product
  const int32_t* w_rowsum;  // RW[N]
  const int32_t* a_rowsum;  // RA[M]
  const float *w_scale, *a_scale, *w_zero, *a_zero;
  __half* out;
  int64_t ldo;
  int32_t layout, M, N, K;
};
cudaError_t launch_zp_epilogue(const ZpArgs& p, cudaStream_t stream);
// ablation (the paper's "Basic" recovery in global memory): out = sum_{i,j} 2^(i+j) parts[i * wbits + j]
cudaError_t launch_recombine_planes(const int32_t* parts, int abits, int wbits, int64_t part_stride, int64_t count,
                                    int32_t* out, cudaStream_t stream);
}  // namespace apt

namespace apt {
// grouped decode GEMM (gemm_grp.cu): up to kGrpMax independent problems (M <= 16, tile-major W, digit-
// view A) in one persistent launch, stream-K over 32-row x 256-K blocks; passed by value (kernel
// parameter space, so a CUDA graph captures the whole group)
constexpr int kGrpMax = 64;
struct GrpProblem {
  CUtensorMap tok;         // activation digit view [M][Kpad] u8, 128 x 16 boxes, 128-byte swizzle
  const uint32_t* wp;      // tile-major weight planes
  int64_t w_pstride;       // words per plane
  const uint8_t* adig;     // activation digits [M][Kpad], kernel K order
  EpilogueArgs e;
  int64_t blk0;            // global index of the problem's first block (tile-major, then K)
  int64_t cost0;           // total cost of the blocks before the problem
  int32_t w_hi;            // worker owning the problem's last block (host-computed: grp_find skips whole
                           // problems with one compare instead of a 64-bit division each)
  const float* w_zero;     // zero points [N] / [M] (fp16 output), nullable
  const float* a_zero;
  void* peers[7];          // epilogue-direct peer stores: the output also goes to these (same offsets)
  int32_t n_peers;
  const float* w_gs;       // group-wise (128) scales [Kpad / 128][N] (GS launches), else null
  const float* a_gs;       // [Kpad / 128][a_gs_ld], nullable (then a_scale per token)
  int64_t a_gs_ld;
  int32_t k_words, nb, tiles, wbits, cost;  // nb = Kpad / 256 blocks per row tile; tiles = ceil(N / 128)
};
constexpr int kGrpMaxWorkers = 1024;
struct GrpArgs {
  int32_t count, workers;  // workers = warps of the grid; workers * max cost <= total_cost
  int64_t total_blocks, total_cost;
  int32_t* partials;       // [workers][2][16 x 32] int32
  uint32_t* tickets;       // [workers], zero before and after the call
  GrpProblem p[kGrpMax];
  uint32_t wstart[kGrpMaxWorkers + 1];  // global index of each worker's first block (host-computed; [workers] = total)
};
int grp_wbmax_class(int wbmax);
int grp_ctas_per_sm(int wbmax, bool gs);
cudaError_t launch_gemm_grp(const GrpArgs& a, int wbmax, int ctas, bool gs, bool peers, cudaStream_t stream);
}  // namespace apt
