// fp64_peak.cu — measured FP64 FMA throughput of this GPU (the FP64 roofline
// denominator bench.py reports next to the HBM one; MEASURED_PEAKS.json has
// no FP64 figure).  Every thread runs 8 independent DFMA chains; best of 5
// launches of 148 x 16 CTAs x 256 threads, CUDA events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o build/fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double));
  const int blocks = nsm * 16, threads = 256, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_loop<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flop = 2.0 * 8.0 * double(iters) * double(blocks) * threads;
  std::printf("{\"fp64_fma_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"how\": \"8 independent DFMA chains per thread, %d x %d threads, %d iterations, best of 5, FMA = 2 flop\"}\n",
              flop / (best * 1e-3) / 1e12, best, nsm, blocks, threads, iters);
  return 0;
}
