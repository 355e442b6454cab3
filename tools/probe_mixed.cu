// Probe: do DFMA (FP64 pipe) and DMMA (tensor DMMA subpipe) share throughput?
// Runs kernels where some warps issue DMMA chains and others DFMA chains, and
// a kernel where each warp interleaves both. Reports combined TF/s.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// mode 0: all DMMA; 1: all DFMA; 2: even warps DMMA, odd DFMA; 3: each warp both (ratio r DFMA per DMMA)
template <int MODE, int R>
__global__ void mixed(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double acc[8][2]; double f[8];
  for (int i = 0; i < 8; i++) { acc[i][0] = acc[i][1] = 0; f[i] = threadIdx.x * 1e-3 + i; }
  double a = threadIdx.x * 1e-3, b = 1e-3, s = 1.0000001, c = 1e-9;
  bool do_mma = MODE == 0 || (MODE == 2 && !(warp & 1)) || MODE == 3;
  bool do_fma = MODE == 1 || (MODE == 2 && (warp & 1)) || MODE == 3;
  for (int it = 0; it < iters; it++) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < 8; i++) dmma(acc[i], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int r = 0; r < R; r++)
#pragma unroll
        for (int i = 0; i < 8; i++) f[i] = fma(f[i], s, c);
    }
  }
  double r = 0;
  for (int i = 0; i < 8; i++) r += acc[i][0] + acc[i][1] + f[i];
  if (r == 12345.0) out[0] = r;
}

template <int MODE, int R>
void run(const char* name, int sms, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 512, blocks = sms * 2, iters = 2048;
  mixed<MODE, R><<<blocks, threads>>>(d, 8); cudaDeviceSynchronize();
  float best = 1e9;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0); mixed<MODE, R><<<blocks, threads>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double warps = (double)blocks * threads / 32;
  double mma_w = MODE == 0 || MODE == 3 ? warps : (MODE == 2 ? warps / 2 : 0);
  double fma_w = MODE == 1 || MODE == 3 ? warps : (MODE == 2 ? warps / 2 : 0);
  double mma_fl = mma_w * iters * 8 * 512.0;          // 8 DMMA x 256 MAC x 2
  double fma_fl = fma_w * 32 * iters * 8 * R * 2.0;
  printf("\"%s\": {\"dmma_tf\": %.2f, \"dfma_tf\": %.2f, \"total_tf\": %.2f},\n", name,
         mma_fl / best / 1e9, fma_fl / best / 1e9, (mma_fl + fma_fl) / best / 1e9);
}

int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\n");
  run<0, 1>("dmma_only", sms, d);
  run<1, 8>("dfma_only", sms, d);
  run<2, 8>("split_warps", sms, d);
  run<3, 2>("interleaved_r2", sms, d);
  run<3, 4>("interleaved_r4", sms, d);
  run<3, 8>("interleaved_r8", sms, d);
  printf("\"end\": 0}\n");
  return 0;
}
