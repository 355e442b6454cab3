// i8gemm_lab.cu -- standalone check + timing of the hand-written tcgen05
// INT8 residue GEMM (paper_2512_23917_b200/csrc/kernels/i8gemm.cu):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/i8gemm_lab.cu -o tools/i8gemm_lab && tools/i8gemm_lab
// Every output of small ragged problems and 4096 sampled outputs of the
// bench-sized ones are compared with a plain int64 dot product mod m.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2512_23917_b200/csrc/kernels/i8gemm.cu"

using namespace tci;

__global__ void fill_rand(int8_t *p, size_t n, uint64_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + i * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = (int8_t)((int)(z % 255) - 127);
  }
}

// reference: sampled (b, m, n) or all when idx == nullptr
__global__ void ref_kernel(const int8_t *A, const int8_t *B, int64_t M, int64_t N, int64_t Kp, int L, int per_mod,
                           const int64_t *idx, int64_t nidx, const int *mods, uint8_t *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nidx) return;
  const int64_t e = idx ? idx[i] : i;
  const int64_t b = e / (M * N), m = (e / N) % M, n = e % N;
  long long acc = 0;
  for (int64_t k = 0; k < Kp; k++) acc += (int)A[(b * M + m) * Kp + k] * (int)B[(b * N + n) * Kp + k];
  const int md = mods[b / per_mod];
  long long r = acc % md;
  if (r < 0) r += md;
  out[i] = (uint8_t)r;
}

static int check(int64_t M, int64_t N, int64_t Kp, int L, int per_mod, bool full, int reps) {
  int8_t *A, *B;
  uint8_t *D, *R;
  int64_t *idx = nullptr;
  int *mods;
  const int hm[16] = {255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193, 1};
  cudaMalloc(&A, (size_t)L * M * Kp);
  cudaMalloc(&B, (size_t)L * N * Kp);
  cudaMalloc(&D, (size_t)L * M * N);
  cudaMalloc(&mods, sizeof hm);
  cudaMemcpy(mods, hm, sizeof hm, cudaMemcpyHostToDevice);
  fill_rand<<<1024, 256>>>(A, (size_t)L * M * Kp, 1);
  fill_rand<<<1024, 256>>>(B, (size_t)L * N * Kp, 2);
  cudaMemset(D, 0xAB, (size_t)L * M * N);
  int64_t nidx = full ? L * M * N : 4096;
  std::vector<int64_t> hidx;
  if (!full) {
    srand(7);
    for (int64_t i = 0; i < nidx; i++) {
      int64_t b = rand() % L, m = (i < 64) ? (i % 2 ? M - 1 : 0) : rand() % M, n = (i % 3 == 0) ? N - 1 : rand() % N;
      hidx.push_back((b * M + m) * N + n);
    }
    cudaMalloc(&idx, nidx * 8);
    cudaMemcpy(idx, hidx.data(), nidx * 8, cudaMemcpyHostToDevice);
  }
  cudaMalloc(&R, nidx);
  cudaError_t e = launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, 0, nullptr);
  if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("run: %s\n", cudaGetErrorString(e)); return 1; }
  ref_kernel<<<(unsigned)((nidx + 127) / 128), 128>>>(A, B, M, N, Kp, L, per_mod, idx, nidx, mods, R);
  cudaDeviceSynchronize();
  std::vector<uint8_t> hr(nidx), hd((size_t)L * M * N);
  cudaMemcpy(hr.data(), R, nidx, cudaMemcpyDeviceToHost);
  cudaMemcpy(hd.data(), D, hd.size(), cudaMemcpyDeviceToHost);
  int64_t bad = 0;
  for (int64_t i = 0; i < nidx; i++) {
    const int64_t eidx = full ? i : hidx[i];
    if (hd[eidx] != hr[i]) {
      if (bad < 5) printf("  mismatch at %lld: got %d want %d\n", (long long)eidx, hd[eidx], hr[i]);
      bad++;
    }
  }
  double ms = 0;
  if (reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, 0, nullptr);
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++) launch_i8gemm(A, B, D, M, N, Kp, L, per_mod, 0, nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t;
    cudaEventElapsedTime(&t, a, b);
    ms = t / reps;
  }
  const double ops = 2.0 * M * N * Kp * L;
  printf("M=%lld N=%lld K=%lld L=%d: %lld/%lld mismatches%s", (long long)M, (long long)N, (long long)Kp, L,
         (long long)bad, (long long)nidx, full ? " (all)" : " (sampled)");
  if (reps) printf("  %.3f ms  %.1f TOPS", ms, ops / ms * 1e-9);
  printf("\n");
  cudaFree(A); cudaFree(B); cudaFree(D); cudaFree(R); cudaFree(mods);
  if (idx) cudaFree(idx);
  return bad != 0;
}

int main(int argc, char **argv) {
  int fails = 0;
  fails += check(256, 256, 128, 1, 1, true, 0);
  fails += check(300, 272, 192, 3, 3, true, 0);
  fails += check(513, 528, 1088, 4, 1, true, 0);
  fails += check(1024, 1024, 4096, 6, 3, false, 3);
  if (argc > 1) {
    fails += check(9216, 16384, 4096, 42, 3, false, 3);    // bench GEMM1 chunk
    fails += check(7680, 4096, 20480, 42, 3, false, 3);    // bench GEMM4 chunk
  }
  printf(fails ? "FAIL\n" : "ALL OK\n");
  return fails;
}
