// Instruction-cache capacity probe: straight-line DFMA bodies of KB kilobytes inside a
// run-time loop, 8 warps per SM (2 CTAs x 4 warps, unsynchronised), time per instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu && ./icache
#include <cstdio>
#include <cuda_runtime.h>

template <int KB>
__global__ void __launch_bounds__(128) body(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < KB * 64; ++i) acc[i % 8] = fma(acc[i % 8], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int KB>
void run(double* out) {
  const int iters = 4096 / KB;  // same instruction count for every size
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  body<KB><<<296, 128>>>(out, iters, 1.0000001, 1e-9);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  body<KB><<<296, 128>>>(out, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double instr = (double)iters * KB * 64;  // per warp
  // 8 warps per SM, 2 per SMSP: DFMA pipe floor = 2 warps x instr x 2 cycles
  printf("KB=%3d  %.3f ms  cycles/instr/warp (at 1.965 GHz) = %.2f\n", KB, ms, ms * 1e-3 * 1.965e9 / instr);
}

int main() {
  double* out;
  cudaMalloc(&out, 296 * 128 * sizeof(double));
  run<8>(out); run<16>(out); run<24>(out); run<28>(out); run<32>(out); run<36>(out); run<40>(out); run<48>(out);
  run<56>(out); run<60>(out); run<64>(out); run<72>(out); run<80>(out); run<96>(out); run<112>(out);
  run<128>(out); run<144>(out); run<160>(out); run<192>(out); run<256>(out);
  return 0;
}
