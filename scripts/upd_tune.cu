// upd_tune.cu — microbenchmark of upd_kernel variants on config-3-sized blocks
// (n = 256^3, s = 16, FP64): the 6-input / 4-output QMR update (10 blocks) and a
// 2-input axpy (3 blocks). Tuning aid only (not part of the product).
#include <cstdio>
#include <cstdlib>

#include "block_kernels.cuh"

using namespace srk;
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int NI, int R, bool STREAM, int MINB>
void run(const UpdArgs& a, size_t smem, int nsm, double bytes, const char* name) {
  auto k = upd_kernel<double, 16, false, NI, R, true, STREAM, MINB>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 48 * 1024));
  const int grid = nsm * occ;
  for (int w = 0; w < 3; ++w) k<<<grid, 256, smem, 0>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int it = 10;
  for (int w = 0; w < it; ++w) k<<<grid, 256, smem, 0>>>(a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= it;
  printf("%-30s occ %d grid %4d  %.3f ms  %.0f GB/s\n", name, occ, grid, ms, bytes / ms / 1e6);
}

__global__ void fill(double* p, long long m, int seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    p[i] = (double)(((i + seed * 7919) * 2654435761ULL) % 1000003) / 1000003.0 - 0.5;
}

int main() {
  const long long n = 256LL * 256 * 256;
  const int s = 16;
  double* blk[8];
  for (int i = 0; i < 8; ++i) {
    CK(cudaMalloc(&blk[i], sizeof(double) * n * s));
    fill<<<1024, 256>>>(blk[i], n * s, i);
  }
  double* yv;
  CK(cudaMalloc(&yv, sizeof(double) * n));
  fill<<<1024, 256>>>(yv, n, 9);
  double *ws, *part;
  CK(cudaMalloc(&ws, sizeof(double) * 64));
  CK(cudaMemset(ws, 0, sizeof(double) * 64));
  CK(cudaMalloc(&part, sizeof(double) * 65536));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const double B = (double)n * s * 8;
  // 6 inputs, 4 outputs (D = eta P + f D; S = eta Pt + f S; X += D; R -= S; ||R||^2)
  UpdArgs a{};
  for (int o = 0; o < MAX_OUT; ++o)
    for (int b = 0; b < MAX_SRC; ++b) a.cf[o][b].kind = CK_NONE;
  a.nin = 6;
  for (int i = 0; i < 6; ++i) a.in[i] = blk[i];
  a.nout = 4;
  a.out[0] = blk[1]; a.out[1] = blk[3]; a.out[2] = blk[4]; a.out[3] = blk[5];
  int cs = 0;
  auto term = [&](int o, int src, int kind) { a.cf[o][src] = Coef{kind, 0, 0, 0, 0}; a.cslot[o][src] = cs; cs += 2; };
  term(0, 0, CK_SCALAR); term(0, 1, CK_SCALAR);
  term(1, 2, CK_SCALAR); term(1, 3, CK_SCALAR);
  term(2, 4, CK_ONE); term(2, SRC_OUT + 0, CK_ONE);
  term(3, 5, CK_ONE); term(3, SRC_OUT + 1, CK_ONE);
  a.cslot_total = cs;
  a.nred = 1; a.red[0] = Red{RED_NORM2, SRC_OUT + 3, -1, nullptr, 0};
  a.ws = ws; a.partials = part; a.pstride = 1; a.n = n; a.s = s; a.vec = 1;
  const size_t smem = cs * 8 + 8 * 8;
  printf("10-block update (%.2f GB)\n", 10 * B / 1e9);
  run<6, 1, false, 2>(a, smem, nsm, 10 * B, "NI6 R1 minb2 (library)");
  run<6, 1, false, 3>(a, smem, nsm, 10 * B, "NI6 R1 minb3");
  run<6, 1, false, 4>(a, smem, nsm, 10 * B, "NI6 R1 minb4");
  run<6, 1, true, 4>(a, smem, nsm, 10 * B, "NI6 R1 stream minb4");
  // 2 inputs, 1 output (P = V - c P)
  UpdArgs b = a;
  for (int o = 0; o < MAX_OUT; ++o)
    for (int q = 0; q < MAX_SRC; ++q) b.cf[o][q].kind = CK_NONE;
  cs = 0;
  b.nin = 2; b.in[0] = blk[0]; b.in[1] = blk[1]; b.nout = 1; b.out[0] = blk[1];
  b.cf[0][0] = Coef{CK_SCALAR, 0, 0, 0, 0}; b.cslot[0][0] = 0;
  b.cf[0][1] = Coef{CK_SCALAR, 0, 1, 0, 0}; b.cslot[0][1] = 2;
  b.cslot_total = 4; b.nred = 0;
  printf("3-block update (%.2f GB)\n", 3 * B / 1e9);
  run<2, 2, false, 2>(b, 64, nsm, 3 * B, "NI2 R2 minb2 (library)");
  run<2, 2, false, 3>(b, 64, nsm, 3 * B, "NI2 R2 minb3");
  run<2, 2, true, 3>(b, 64, nsm, 3 * B, "NI2 R2 stream minb3");
  run<2, 2, false, 4>(b, 64, nsm, 3 * B, "NI2 R2 minb4");
  run<2, 4, false, 3>(b, 64, nsm, 3 * B, "NI2 R4 minb3");
  run<2, 1, false, 4>(b, 64, nsm, 3 * B, "NI2 R1 minb4");
  // 2 inputs, 1 output with ||out||^2 and sum_i conj(w_i) out_i (eGl-QMR V~ update)
  UpdArgs v = b;
  v.nred = 2;
  v.pstride = 17;
  v.red[0] = Red{RED_NORM2, SRC_OUT + 0, -1, nullptr, 0};
  v.red[1] = Red{RED_SUMVEC, SRC_OUT + 0, -1, yv, 1};
  printf("3-block update + NORM2 + SUMVEC (%.2f GB + n-vector)\n", 3 * B / 1e9);
  run<2, 2, false, 4>(v, 64 + 8 * 64, nsm, 3 * B, "red NI2 R2 minb4 (library)");
  run<2, 2, false, 3>(v, 64 + 8 * 64, nsm, 3 * B, "red NI2 R2 minb3");
  run<2, 2, false, 2>(v, 64 + 8 * 64, nsm, 3 * B, "red NI2 R2 minb2");
  run<2, 1, false, 4>(v, 64 + 8 * 64, nsm, 3 * B, "red NI2 R1 minb4");
  run<2, 4, false, 2>(v, 64 + 8 * 64, nsm, 3 * B, "red NI2 R4 minb2");
  run<2, 2, false, 4>(b, 64, nsm, 3 * B, "nored NI2 R2 minb4 (library)");
  UpdArgs v1 = v; v1.nred = 1;
  run<2, 2, false, 4>(v1, 64 + 8 * 64, nsm, 3 * B, "NORM2 only NI2 R2 minb4");
  UpdArgs v2 = v; v2.nred = 1; v2.red[0] = v.red[1];
  run<2, 2, false, 4>(v2, 64 + 8 * 64, nsm, 3 * B, "SUMVEC only NI2 R2 minb4");
  UpdArgs v3 = v; v3.red[1] = Red{RED_NORM2, SRC_OUT + 0, -1, nullptr, 1};
  run<2, 2, false, 4>(v3, 64 + 8 * 64, nsm, 3 * B, "NORM2 x2 NI2 R2 minb4");
  // 1 input (V = c Vt)
  UpdArgs c1 = b;
  c1.nin = 1; c1.cf[0][1].kind = CK_NONE;
  printf("2-block update (%.2f GB)\n", 2 * B / 1e9);
  run<1, 4, false, 2>(c1, 64, nsm, 2 * B, "NI1 R4 minb2 (library)");
  run<1, 4, false, 3>(c1, 64, nsm, 2 * B, "NI1 R4 minb3");
  run<1, 2, false, 4>(c1, 64, nsm, 2 * B, "NI1 R2 minb4");
  run<1, 4, false, 4>(c1, 64, nsm, 2 * B, "NI1 R4 minb4");
  return 0;
}
