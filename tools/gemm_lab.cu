// gemm_lab.cu -- standalone A/B harness for gemm_dmma.cu variants (not part of
// the library). Times C = A.B for the H_eff GEMM shapes with CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/gemm_lab tools/gemm_lab.cu
#ifdef NODADD
#define TCI_LAB_SUM(x, y) (x)
#endif
#include "../paper_2512_23917_b200/csrc/kernels/gemm_dmma.cu"
#include <vector>
#include <cstdio>

namespace tci { cudaError_t launch_gemm_f32(const GemmProblem &, cudaStream_t, int64_t *) { return cudaErrorNotSupported; } }
using namespace tci;

__global__ void fill(double* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed + i) * 0x9E3779B97F4A7C15ull; z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    p[i] = (double)(z >> 11) * 0x1.0p-52 - 1.0;
  }
}

template <class C>
double time_cfg(const GemmProblem& p, int reps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  run<C>(p, 0, nullptr); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(e0); run<C>(p, 0, nullptr); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return best / 1e3;
}

int main(int argc, char** argv) {
  // GEMM4 of the target: M = 16384 (b p q), K = 20480 (c x), N = 4096; A K-major, B N-major
  int64_t M = 16384, N = 4096, K = 20480;
  if (argc > 3) { M = atoll(argv[1]); N = atoll(argv[2]); K = atoll(argv[3]); }
  double *A, *B, *Cm;
  cudaMalloc(&A, M * K * 16); cudaMalloc(&B, K * N * 16); cudaMalloc(&Cm, M * N * 16);
  fill<<<1024, 256>>>(A, M * K * 2, 1); fill<<<1024, 256>>>(B, K * N * 2, 2);
  GemmProblem p{}; p.dtype = TCI_C128; p.M = M; p.N = N; p.K = K;
  p.A = A; p.a_sm = K; p.a_sk = 1; p.B = B; p.b_sk = N; p.b_sn = 1; p.C = Cm; p.c_sm = N;
  const double F = 8.0 * M * N * K;
  auto rep = [&](const char* name, double t) { printf("%-40s %8.2f ms  %6.2f TF/s (alg)\n", name, t * 1e3, F / t / 1e12); };
  rep("3M  64x64 bk8 w32x16 s6", time_cfg<Cfg<kCplx3M, 64, 64, 8, 32, 16, 6, true, false, 1>>(p, 3));
  rep("3MS 64x64 bk8 w32x16 s6", time_cfg<Cfg<kCplx3MS, 64, 64, 8, 32, 16, 6, true, false, 1>>(p, 3));
  rep("3MS 64x64 bk16 w32x16 s4", time_cfg<Cfg<kCplx3MS, 64, 64, 16, 32, 16, 4, true, false, 1>>(p, 3));
  rep("3MS 64x64 bk8 w32x16 s5", time_cfg<Cfg<kCplx3MS, 64, 64, 8, 32, 16, 5, true, false, 1>>(p, 3));
  rep("3MS 64x64 bk8 w16x32 s6", time_cfg<Cfg<kCplx3MS, 64, 64, 8, 16, 32, 6, true, false, 1>>(p, 3));
  p.A = A; p.a_sm = 1; p.a_sk = M;   // GEMM1-like: A M-major
  rep("[A M-major] 3M  bk8 s6", time_cfg<Cfg<kCplx3M, 64, 64, 8, 32, 16, 6, false, false, 1>>(p, 3));
  rep("[A M-major] 3MS bk8 s6", time_cfg<Cfg<kCplx3MS, 64, 64, 8, 32, 16, 6, false, false, 1>>(p, 3));
  rep("[A M-major] 3MS bk16 s4", time_cfg<Cfg<kCplx3MS, 64, 64, 16, 32, 16, 4, false, false, 1>>(p, 3));
  return 0;
}
