// kernels.h — launch interfaces between the C-ABI shim (apt.cu) and the kernels.
#pragma once
#include <cstdint>
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
};
cudaError_t launch_pack(const PackArgs& p, int bits, cudaStream_t stream);

struct MmaArgs {
  const uint32_t* wp;      // weight planes [wbits][N][k_words]
  int64_t w_pstride;       // N * k_words
  const uint32_t* ap;      // activation planes [abits][M][k_words]
  int64_t a_pstride;       // M * k_words
  int32_t k_words;
  int32_t abits;
  int32_t kw_per_split;    // multiple of 8
  EpilogueArgs e;
};
cudaError_t launch_gemm_mma(const MmaArgs& p, int wbits, int bn, int split, cudaStream_t stream);
size_t mma_smem_bytes(int bn, int split);

}  // namespace apt

namespace apt {
struct TcArgs {
  const uint32_t* wp;      // weight planes [wbits][N][k_words]
  int64_t w_pstride;       // N * k_words
  const uint32_t* ap;      // activation planes [abits][M][k_words]
  int64_t a_pstride;       // M * k_words
  int32_t k_words;
  int32_t abits;
  EpilogueArgs e;
};
cudaError_t launch_gemm_tc(const TcArgs& p, int wbits, int bn, int stages, void* workspace, cudaStream_t stream);
int tc_stages(int wbits, int bn);
size_t tc_workspace_bytes(int M, int k_words);
}  // namespace apt
