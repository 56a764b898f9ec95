// PDL chain floor: per-launch time of back-to-back launches (CUDA graph, programmatic dependent launch)
// of kernels that do (a) nothing but launch_dependents + wait + one store, (b) the same plus one
// dependent L2 load after the wait, for a few grid shapes.  Separates the per-launch cost of the
// stream/PDL machinery from a GEMM's own critical path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_floor chain_floor.cu && ./chain_floor
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* out, const int* in, int mode) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int v = 0;
  if (mode >= 1) v = __ldcg(in + (blockIdx.x * 37 + threadIdx.x) % 4096);
  if (mode >= 2) v += __ldcg(in + (v & 4095));
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

int main() {
  int *out, *in;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&in, 1 << 20);
  cudaMemset(in, 0, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  printf("{\"probe\": \"chain_floor\", \"rows\": [\n");
  bool first = true;
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int mode = 0; mode < 3; ++mode)
      for (int ctas : {128, 296, 1024})
        for (int threads : {128, 512}) {
          const int L = 32;
          cudaGraph_t g;
          cudaGraphExec_t ge;
          cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
          for (int i = 0; i < L; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctas);
            cfg.blockDim = dim3(threads);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = pdl;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_empty, out, in, mode);
          }
          cudaStreamEndCapture(s, &g);
          cudaGraphInstantiate(&ge, g, 0);
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, s);
          float best = 1e9;
          for (int r = 0; r < 10; ++r) {
            cudaEventRecord(e0, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaStreamSynchronize(s);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
          }
          printf("%s{\"pdl\": %d, \"loads_after_wait\": %d, \"ctas\": %d, \"threads\": %d, \"us_per_launch\": %.3f}\n",
                 first ? "" : ",", pdl, mode, ctas, threads, best * 1e3 / L);
          first = false;
          cudaGraphExecDestroy(ge);
          cudaGraphDestroy(g);
        }
  printf("]}\n");
  return 0;
}
