// Standalone timing of the tcgen05 update GEMM (k_gemm_tc) at the c2-gcn layer shapes,
// outside the engine: A image / weights random, CUDA events over R launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2603_20622_b200/csrc \
//        tools/gemm_micro.cu -L paper_2603_20622_b200 -lrtec -o gpurun_out/gemm_micro
// usage: gemm_micro M d_in d_out fused(0/1) [reps]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "gemm_tc.cuh"
#include "rtec.h"

__global__ void fill(float* p, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = static_cast<uint32_t>(i) * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xFFFFFF) / 16777216.0f - 0.5f;
  }
}
__global__ void fill_i(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v + (i & 7);
}

int main(int argc, char** argv) {
  int64_t M = argc > 1 ? atoll(argv[1]) : 2000000;
  int d_in = argc > 2 ? atoi(argv[2]) : 256, d_out = argc > 3 ? atoi(argv[3]) : 256;
  int fused = argc > 4 ? atoi(argv[4]) : 0, reps = argc > 5 ? atoi(argv[5]) : 20;
  int nkb = rtec::tc_nkb_of(d_in), npad = rtec::tc_npad_of(d_out);
  int64_t tiles = (M + 127) / 128;
  float *A, *W, *Bhi, *Blo, *Y, *D = nullptr;
  int32_t* deg = nullptr;
  cudaMalloc(&A, tiles * nkb * 128 * 32 * 4);
  cudaMalloc(&W, (size_t)d_out * d_in * 4);
  cudaMalloc(&Bhi, (size_t)nkb * npad * 32 * 4);
  cudaMalloc(&Blo, (size_t)nkb * npad * 32 * 4);
  cudaMalloc(&Y, M * d_out * 4);
  fill<<<1184, 256>>>(A, tiles * nkb * 128 * 32, 1);
  fill<<<1184, 256>>>(W, (int64_t)d_out * d_in, 2);
  fill<<<1184, 256>>>(Y, M * d_out, 3);
  rtec_gemm_prepare_weights(W, d_in, d_out, Bhi, Blo, nullptr);
  rtec::TcArgs g{};
  g.A = A; g.Bhi = Bhi; g.Blo = Blo; g.nkb = nkb; g.npad = npad; g.d_out = d_out;
  g.max_rows = M; g.act = 1; g.Y = Y; g.ldy = d_out;
  if (fused) {
    cudaMalloc(&D, M * d_out * 4);
    cudaMalloc(&deg, M * 4);
    fill_i<<<1184, 256>>>(deg, M, 3);
    g.delta_next = D; g.deg_new = deg; g.deg_old = deg; g.coeff_gcn = 1; g.deg_off = 1.f;
  }
  // L2 flush buffer
  float* fl; cudaMalloc(&fl, 256ull << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) rtec::gemm_tc_launch(g, 0);
  float tot = 0;
  for (int i = 0; i < reps; ++i) {
    cudaMemsetAsync(fl, i, 256ull << 20);
    cudaEventRecord(e0);
    rtec::gemm_tc_launch(g, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); tot += ms;
  }
  cudaError_t err = cudaDeviceSynchronize();
  double ms = tot / reps;
  double fl3 = 2.0 * M * d_in * d_out * 3;
  // MMA floor (B300 microarch model: 128*N/256 cycles per K=8 tf32 dispatch at cta_group::1)
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double disp_cyc = (double)tiles * nkb * 4 * 3 * (128.0 * npad / 256.0) / sms;
  printf("{\"M\": %lld, \"d_in\": %d, \"d_out\": %d, \"fused\": %d, \"ms\": %.4f, \"tf32x3_TFLOPs\": %.1f, "
         "\"mma_floor_ms\": %.4f, \"clk_mhz\": %d, \"err\": \"%s\"}\n",
         (long long)M, d_in, d_out, fused, ms, fl3 / ms / 1e9, disp_cyc / (clk * 1e3) * 1e3, clk / 1000,
         cudaGetErrorString(err));
  return 0;
}
