// spmm_tune.cu — microbenchmark of spmm_kernel variants on the config-3 operator
// (256^3 7-point stencil, s = 16, FP64) with the eGl SUMVEC epilogue. Builds the
// CSR on the host, times each variant with CUDA events (warm, 20 launches), and
// prints the achieved algorithmic GB/s. Tuning aid only (not part of the product).
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_1504_04395_b200/csrc \
//        -I scripts scripts/spmm_tune.cu -o scripts/spmm_tune -lcuda
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <vector>

#include <cuda.h>

#include "spmm_tma.cuh"  // scripts/ (experiment, not part of the library)

using namespace srk;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int R, int BC, bool YPRE, int MINB, int BATCH = 0, int PD = 1>
float run(const SpmmArgs& a0, int nsm, double bytes, const char* name) {
  auto k = spmm_kernel<double, 16, false, R, true, BC, YPRE, MINB, BATCH, PD>;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 8 * 8 * 2));
  const int grid = nsm * occ;
  SpmmArgs a = a0;
  for (int w = 0; w < 3; ++w) k<<<grid, 256, 8 * 8 * 2, 0>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) k<<<grid, 256, 8 * 8 * 2, 0>>>(a);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= it;
  printf("%-34s occ %d grid %5d  %.3f ms  %.0f GB/s\n", name, occ, grid, ms, bytes / ms / 1e6);
  return ms;
}

TmaDesc make_map(double* P, long long n, int s, int boxrows) {
  TmaDesc d;
  cuuint64_t dims[2] = {(cuuint64_t)s, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)s * 8};
  cuuint32_t box[2] = {(cuuint32_t)s, (cuuint32_t)boxrows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(reinterpret_cast<CUtensorMap*>(&d), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed %d\n", (int)r); exit(1); }
  return d;
}

template <int EMAX, int NST, int NP>
float run_tma(const SpmmArgs& a, const TmaDesc& map, int nsm, double bytes, const char* name) {
  auto k = spmm_tma_kernel<double, 16, false, EMAX, NST, NP>;
  using C = TmaCfg<double, 16, false, EMAX, NST, NP>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, C::NT, C::SMEM));
  const int grid = nsm * occ;
  for (int w = 0; w < 3; ++w) k<<<grid, C::NT, C::SMEM, 0>>>(a, map);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) k<<<grid, C::NT, C::SMEM, 0>>>(a, map);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= it;
  printf("%-34s occ %d grid %5d  %.3f ms  %.0f GB/s  (smem %d)\n", name, occ, grid, ms, bytes / ms / 1e6, C::SMEM);
  return ms;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 256;
  const long long n = (long long)m * m * m;
  const int s = 16;
  std::vector<int> rp(n + 1);
  std::vector<int> ci;
  std::vector<double> va;
  ci.reserve(7 * n);
  va.reserve(7 * n);
  const double h = 1.0 / (m + 1), c[3] = {50, 30, 10};
  long long strides[3] = {1, m, (long long)m * m};
  for (long long i = 0; i < n; ++i) {
    rp[i] = (int)ci.size();
    const int x = i % m, y = (i / m) % m, z = i / ((long long)m * m);
    const int co[3] = {x, y, z};
    // ascending columns: -z, -y, -x, diag, +x, +y, +z
    for (int d = 2; d >= 0; --d)
      if (co[d] > 0) { ci.push_back((int)(i - strides[d])); va.push_back(-1.0 - c[d] * h / 2); }
    ci.push_back((int)i);
    va.push_back(6.0);
    for (int d = 0; d < 3; ++d)
      if (co[d] < m - 1) { ci.push_back((int)(i + strides[d])); va.push_back(-1.0 + c[d] * h / 2); }
  }
  rp[n] = (int)ci.size();
  const long long nnz = ci.size();
  int *drp, *dci;
  double *dva, *P, *Q, *y, *part;
  CK(cudaMalloc(&drp, sizeof(int) * (n + 5)));
  CK(cudaMalloc(&dci, sizeof(int) * (nnz + 4)));
  CK(cudaMemset(dci, 0, sizeof(int) * (nnz + 4)));
  CK(cudaMalloc(&dva, sizeof(double) * (nnz + 2)));
  CK(cudaMemset(dva, 0, sizeof(double) * (nnz + 2)));
  CK(cudaMalloc(&P, sizeof(double) * n * s));
  CK(cudaMalloc(&Q, sizeof(double) * n * s));
  CK(cudaMalloc(&y, sizeof(double) * n));
  CK(cudaMalloc(&part, sizeof(double) * 4096));
  CK(cudaMemcpy(drp, rp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dva, va.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemset(P, 0, sizeof(double) * n * s));
  CK(cudaMemset(y, 0, sizeof(double) * n));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  SpmmArgs a{};
  a.row_ptr = drp; a.col_idx = dci; a.val = dva; a.P = P; a.Q = Q; a.n = n; a.s = s; a.vec = 1;
  a.nred = 1; a.red[0].mode = RED_SUMVEC; a.red[0].yext = y; a.red[0].poff = 0; a.partials = part; a.pstride = 1;
  const double bytes = (n + 1) * 4.0 + nnz * 12.0 + 2.0 * n * s * 8 + n * 8.0;
  printf("n %lld nnz %lld algorithmic %.3f GB\n", n, nnz, bytes / 1e9);
  const int boxrows = argc > 2 ? atoi(argv[2]) : 1;
  {
    std::vector<double> hp(n * s);
    for (long long i = 0; i < n * s; ++i) hp[i] = (double)((i * 2654435761ULL) % 1000003) / 1000003.0 - 0.5;
    CK(cudaMemcpy(P, hp.data(), sizeof(double) * n * s, cudaMemcpyHostToDevice));
    std::vector<double> hy(n);
    for (long long i = 0; i < n; ++i) hy[i] = (double)((i * 40503ULL) % 1009) / 1009.0;
    CK(cudaMemcpy(y, hy.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  }
  TmaDesc map = make_map(P, n, s, boxrows);
  {
    double* Q2;
    double* part2;
    CK(cudaMalloc(&Q2, sizeof(double) * n * s));
    CK(cudaMalloc(&part2, sizeof(double) * 4096));
    CK(cudaMemset(Q2, 0, sizeof(double) * n * s));
    SpmmArgs b = a; b.Q = Q2; b.partials = part2;
    using C = TmaCfg<double, 16, false, 228, 3, 4>;
    CK(cudaFuncSetAttribute(spmm_tma_kernel<double, 16, false, 228, 3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    spmm_kernel<double, 16, false, 2, true><<<296, 256, 8 * 8 * 2, 0>>>(a);
    spmm_tma_kernel<double, 16, false, 228, 3, 4><<<148, C::NT, C::SMEM, 0>>>(b, map);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<double> h1(n * s), h2(n * s), p1(296), p2(148);
    CK(cudaMemcpy(h1.data(), Q, sizeof(double) * n * s, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), Q2, sizeof(double) * n * s, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(p1.data(), part, sizeof(double) * 296, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(p2.data(), part2, sizeof(double) * 148, cudaMemcpyDeviceToHost));
    double md = 0, s1 = 0, s2 = 0;
    for (long long i = 0; i < n * s; ++i) md = fmax(md, fabs(h1[i] - h2[i]));
    for (int i = 0; i < 296; ++i) s1 += p1[i];
    for (int i = 0; i < 148; ++i) s2 += p2[i];
    printf("tma vs library: max |dQ| = %.3e   sumvec %.15e vs %.15e\n", md, s1, s2);
  }
  run<2, 8, true, 2, 8, 1>(a, nsm, bytes, "R2 minb2 batch8 (library)");
  run<2, 8, true, 3, 8, 1>(a, nsm, bytes, "R2 minb3 batch8");
  run<2, 8, true, 3, 4, 1>(a, nsm, bytes, "R2 minb3 batch4");
  run<2, 8, true, 4, 4, 1>(a, nsm, bytes, "R2 minb4 batch4");
  run<1, 8, true, 3, 8, 1>(a, nsm, bytes, "R1 minb3 batch8");
  run<1, 8, true, 4, 8, 1>(a, nsm, bytes, "R1 minb4 batch8");
  run<1, 16, true, 4, 8, 1>(a, nsm, bytes, "R1 BC16 minb4 batch8");
  run<2, 2, true, 2, 8, 1>(a, nsm, bytes, "R2 BC2 minb2 batch8");
  run<2, 4, true, 2, 8, 1>(a, nsm, bytes, "R2 BC4 minb2 batch8");
  run<2, 16, true, 2, 8, 1>(a, nsm, bytes, "R2 BC16 minb2 batch8");
  run<2, 32, true, 2, 8, 1>(a, nsm, bytes, "R2 BC32 minb2 batch8");
  run<2, 64, true, 2, 8, 1>(a, nsm, bytes, "R2 BC64 minb2 batch8");
  run<2, 8, true, 2, 8, 2>(a, nsm, bytes, "R2 minb2 batch8 PD2");
  run<2, 8, true, 2, 8, 1>(a, nsm, bytes, "R2 minb2 batch8 (repeat)");
  return 0;
}
