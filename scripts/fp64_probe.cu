// fp64_probe.cu — measured FP64 peaks of this B200: DFMA (CUDA cores) and DMMA
// (mma.sync.m8n8k4.f64 tensor cores), register-resident independent chains.
// Tuning aid for the s x s Gram design; prints TFLOP/s.
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int iters = 20000;
    dfma_loop<<<nsm, 32 * warps>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<nsm, 32 * warps>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 16 * iters * 32.0 * warps * nsm;
    printf("DFMA  warps/SM %2d: %.2f TFLOP/s\n", warps, fl / ms / 1e9);
    dmma_loop<<<nsm, 32 * warps>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<<<nsm, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double fm = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * nsm;
    printf("DMMA  warps/SM %2d: %.2f TFLOP/s\n", warps, fm / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
