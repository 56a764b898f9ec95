/* CPU oracle: plain int64 GEMM on signed integer codes (C, OpenMP).
 *
 * TEST INFRASTRUCTURE ONLY.  Built by __graft_entry__.build() into
 * oracle/liboracle.so; loaded only by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs.  Shares no code with the
 * CUDA product path.
 *
 * Computes the plain definition the north_star names ("a plain CPU int64 GEMM
 * on the unpacked signed integers"):
 *     Y[m][n] = sum_{k<K} A[m][k] * W[n][k]          (int64 accumulation)
 * Both operands K-contiguous (reading Q2).  Triple loop, K innermost, no
 * blocking; rows of Y are distributed over OpenMP threads.
 * Pinned in tests/test_oracle.py against numpy int64 matmul and a Python
 * big-int triple loop.
 */
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int apt_oracle_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void apt_oracle_gemm_i64(const int8_t* A, int64_t lda, const int8_t* W, int64_t ldw,
                         int64_t* Y, int64_t ldy, int32_t M, int32_t N, int32_t K) {
#pragma omp parallel for schedule(static)
  for (int32_t m = 0; m < M; ++m) {
    for (int32_t n = 0; n < N; ++n) {
      int64_t acc = 0;
      for (int32_t k = 0; k < K; ++k) acc += (int64_t)A[(int64_t)m * lda + k] * (int64_t)W[(int64_t)n * ldw + k];
      Y[(int64_t)m * ldy + n] = acc;
    }
  }
}
