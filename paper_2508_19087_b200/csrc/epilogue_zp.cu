// epilogue_zp.cu — fp16 output with zero points as a second pass.
//
// Linear quantization with zero points on both operands: x = a_scale x_hat + a_zero,
// W = w_scale w_hat + w_zero, so
//   sum_k x W = as ws Y + az ws RW[n] + as wz RA[m] + K az wz.
// Folding the three rank-1 terms into the GEMM kernels' shared epilogue cost the 128 x 256 prefill
// tile 25% even when no zero points were passed (reading Q10), so the GEMM writes the exact
// int32 Y (signed product) into the caller's workspace and this elementwise kernel evaluates
//   v = ((float)Y * ws) * as;  v += ((float)RW * ws) * az;  v += ((float)RA * as) * wz;  v += ((float)K * az) * wz
// in fp32 in that order and rounds once to fp16.  RW, RA < 2^24 are exact in fp32.  The GEMMs without
// zero points are untouched.
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "sync.cuh"

namespace apt {

__global__ void __launch_bounds__(256) zp_epilogue_kernel(ZpArgs p) {
  pdl_launch_dependents();
  pdl_wait();  // Y comes from the GEMM just before
  const int64_t total = (int64_t)p.M * p.N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / p.N), n = (int)(i % p.N);
    const float ws = __ldg(p.w_scale + n);
    const float as = p.a_scale ? __ldg(p.a_scale + m) : 1.f;
    const float az = p.a_zero ? __ldg(p.a_zero + m) : 0.f;
    const float wz = p.w_zero ? __ldg(p.w_zero + n) : 0.f;
    // every product and sum rounded on its own (no FMA contraction): the documented fp32 order, and the
    // same bits as the grouped kernel's fused zero-point epilogue
    float v = __fmul_rn(__fmul_rn((float)__ldg(p.y + i), ws), as);
    v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)__ldg(p.w_rowsum + n), ws), az));
    v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)__ldg(p.a_rowsum + m), as), wz));
    v = __fadd_rn(v, __fmul_rn(__fmul_rn((float)p.K, az), wz));
    const int64_t off = p.layout == 0 ? (int64_t)m * p.ldo + n : (int64_t)n * p.ldo + m;
    p.out[off] = __float2half_rn(v);
  }
}

cudaError_t launch_zp_epilogue(const ZpArgs& p, cudaStream_t stream) {
  const int64_t total = (int64_t)p.M * p.N;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_pdl(zp_epilogue_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, dim3(1, 1, 1), p);
}

}  // namespace apt

// ---------------------------------------------------------------------------------------------
// Recovery in global memory (the paper's "Basic" design, ablation §6.5):
// the p_a x p_w plane-pair products Y^(i,j) (int32, each from a 1-bit x 1-bit GEMM) are
// recombined in HBM by the shift-add of P:228,  out = sum_{i<p_a, j<p_w} 2^(i+j) Y^(i,j)  (mod 2^32).
// The product path never takes this route (its shift-add is folded into the operand rebuild); this
// kernel exists to measure what that folding saves.
namespace apt {
__global__ void __launch_bounds__(256) recombine_planes_kernel(const int32_t* __restrict__ parts, int32_t abits,
                                                               int32_t wbits, int64_t part_stride, int64_t count,
                                                               int32_t* __restrict__ out) {
  pdl_launch_dependents();
  pdl_wait();  // the plane products come from the GEMMs just before
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int i = 0; i < abits; ++i)
      for (int j = 0; j < wbits; ++j)
        acc += (uint32_t)__ldg(parts + (int64_t)(i * wbits + j) * part_stride + e) << (i + j);
    out[e] = (int32_t)acc;
  }
}

cudaError_t launch_recombine_planes(const int32_t* parts, int abits, int wbits, int64_t part_stride, int64_t count,
                                    int32_t* out, cudaStream_t stream) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return launch_pdl(recombine_planes_kernel, dim3((unsigned)blocks), dim3(256), 0, stream, dim3(1, 1, 1), parts,
                    abits, wbits, part_stride, count, out);
}
}  // namespace apt
