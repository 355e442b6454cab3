// ozaki_lab.cu -- standalone check of the Ozaki-II INT8 complex GEMM against
// the DMMA 3M GEMM (not part of the library): rel. Frobenius difference and time.
#include "../paper_2512_23917_b200/csrc/kernels/gemm_dmma.cu"
#include "../paper_2512_23917_b200/csrc/kernels/ozaki.cu"
#include <cstdio>
#include <vector>
namespace tci { cudaError_t launch_gemm_f32(const GemmProblem &, cudaStream_t, int64_t *) { return cudaErrorNotSupported; } }
using namespace tci;

__global__ void fillz(double* p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = (seed + i) * 0x9E3779B97F4A7C15ull; z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    p[i] = (double)(z >> 11) * 0x1.0p-52 - 1.0;
  }
}
__global__ void diffnorm(const double* a, const double* b, size_t n, double* out) {
  __shared__ double s1[256], s2[256];
  double d = 0, r = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    d += (a[i] - b[i]) * (a[i] - b[i]); r += b[i] * b[i]; }
  s1[threadIdx.x] = d; s2[threadIdx.x] = r; __syncthreads();
  for (int s = 128; s; s >>= 1) { if (threadIdx.x < s) { s1[threadIdx.x] += s1[threadIdx.x + s]; s2[threadIdx.x] += s2[threadIdx.x + s]; } __syncthreads(); }
  if (threadIdx.x == 0) { atomicAdd(out, s1[0]); atomicAdd(out + 1, s2[0]); }
}

int main(int argc, char** argv) {
  struct Sh { int64_t M, N, K; bool ak; } shapes[] = {{16384, 4096, 20480, true}, {20480, 16384, 4096, false}, {300, 77, 1000, true}};
  for (auto sh : shapes) {
    int64_t M = sh.M, N = sh.N, K = sh.K;
    double *A, *B, *C1, *C2, *acc; void* ws;
    cudaMalloc(&A, M * K * 16); cudaMalloc(&B, K * N * 16); cudaMalloc(&C1, M * N * 16); cudaMalloc(&C2, M * N * 16);
    cudaMalloc(&acc, 16);
    fillz<<<1024, 256>>>(A, M * K * 2, 1); fillz<<<1024, 256>>>(B, K * N * 2, 2);
    GemmProblem p{}; p.dtype = TCI_C128; p.M = M; p.N = N; p.K = K;
    p.A = A; if (sh.ak) { p.a_sm = K; p.a_sk = 1; } else { p.a_sm = 1; p.a_sk = M; }
    p.B = B; p.b_sk = N; p.b_sn = 1; p.C = C1; p.c_sm = N;
    size_t wsb = ozaki_workspace_bytes(M, N, K);
    cudaMalloc(&ws, wsb);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float t_dm = 0, t_oz = 0;
    auto tm = [&](auto f) { f(); cudaDeviceSynchronize(); float best = 1e30f; for (int r = 0; r < 3; r++) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; } return best; };
    if (sh.ak) t_dm = tm([&] { run<Z3Cfg<true, false>>(p, 0, nullptr); });
    else t_dm = tm([&] { run<Z3Cfg<false, false>>(p, 0, nullptr); });
    GemmProblem q = p; q.C = C2;
    cudaError_t err = cudaSuccess;
    t_oz = tm([&] { err = launch_ozaki_zgemm(q, ws, wsb, 0, nullptr); });
    if (err) printf("ozaki err %s\n", cudaGetErrorString(err));
    cudaError_t e = cudaDeviceSynchronize(); if (e) printf("cuda %s\n", cudaGetErrorString(e));
    cudaMemset(acc, 0, 16);
    diffnorm<<<1024, 256>>>(C2, C1, M * N * 2, acc);
    double h[2]; cudaMemcpy(h, acc, 16, cudaMemcpyDeviceToHost);
    const double F = 8.0 * M * N * K;
    printf("M=%lld N=%lld K=%lld A_K=%d: DMMA3M %.2f ms (%.1f TF/s) | Ozaki %.2f ms (%.1f TF/s) | rel diff %.3e | ws %.2f GB\n",
           (long long)M, (long long)N, (long long)K, (int)sh.ak, t_dm, F / t_dm / 1e9, t_oz, F / t_oz / 1e9, sqrt(h[0] / h[1]), wsb / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C1); cudaFree(C2); cudaFree(ws); cudaFree(acc);
  }
  return 0;
}
