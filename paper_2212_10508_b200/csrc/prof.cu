// Live per-stage timing (CUDA events on the launching stream) and an FP64
// DFMA peak probe: the roofline numerator/denominator of bench.py.
#include <vector>

#include "pl_common.cuh"

namespace pl {

struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};

struct Prof {
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};

static thread_local Prof g_prof;

bool prof_on() { return g_prof.on; }

void prof_mark(cudaStream_t st, int stage, bool begin) {
  if (!g_prof.on) return;
  cudaEvent_t e = g_prof.get();
  cudaEventRecord(e, st);
  if (begin) {
    g_prof.recs.push_back({stage, e, nullptr});
  } else {
    for (auto it = g_prof.recs.rbegin(); it != g_prof.recs.rend(); ++it)
      if (it->stage == stage && it->b == nullptr) {
        it->b = e;
        break;
      }
  }
}

__global__ void k_dfma_peak(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double m = 0.999999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// FP64 tensor-core (DMMA) throughput: mma.sync m8n8k4 f64, 8 independent
// accumulator tiles per warp (256 FMA per instruction and warp)
__global__ void k_dmma_peak(double* out, int iters) {
  const int lane = threadIdx.x & 31;
  const double a = 1.0 + lane * 1e-9, b = 0.999999 - lane * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = t * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace pl

extern "C" {

int pl_prof_begin(pl_ctx* ctx) {
  if (!ctx) return pl::fail(PL_EARG, "ctx is NULL");
  pl::g_prof.on = true;
  pl::g_prof.recs.clear();
  pl::g_prof.used = 0;
  return PL_OK;
}

// h_ms[s] = summed kernel time of stage s, h_n[s] = launches (s < n_stages)
int pl_prof_end(pl_ctx* ctx, int n_stages, double* h_ms, int64_t* h_n) {
  if (!ctx || !h_ms || !h_n) return pl::fail(PL_EARG, "NULL argument");
  PL_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int s = 0; s < n_stages; ++s) {
    h_ms[s] = 0.0;
    h_n[s] = 0;
  }
  for (auto& r : pl::g_prof.recs) {
    if (!r.b || r.stage < 0 || r.stage >= n_stages) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    h_ms[r.stage] += ms;
    h_n[r.stage] += 1;
  }
  pl::g_prof.on = false;
  pl::g_prof.recs.clear();
  pl::g_prof.used = 0;
  return PL_OK;
}

// measured dense FP64 FMA throughput (TFLOP/s) of this device
int pl_fp64_peak(pl_ctx* ctx, double* h_tflops) {
  if (!ctx || !h_tflops) return pl::fail(PL_EARG, "NULL argument");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  PL_CUDA(cudaMalloc(&out, sizeof(double)));
  const int threads = 256, blocks = sms * 8, iters = 4096;
  pl::k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, ctx->stream);
  pl::k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(out, iters);
  cudaEventRecord(b, ctx->stream);
  PL_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  *h_tflops = flops / (ms * 1e-3) / 1e12;
  return PL_OK;
}

// measured FP64 tensor-core (DMMA m8n8k4) throughput of this device (TFLOP/s)
int pl_dmma_peak(pl_ctx* ctx, double* h_tflops) {
  if (!ctx || !h_tflops) return pl::fail(PL_EARG, "NULL argument");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  PL_CUDA(cudaMalloc(&out, sizeof(double)));
  const int threads = 256, blocks = sms * 4, iters = 2048;
  pl::k_dmma_peak<<<blocks, threads, 0, ctx->stream>>>(out, 32);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, ctx->stream);
  pl::k_dmma_peak<<<blocks, threads, 0, ctx->stream>>>(out, iters);
  cudaEventRecord(b, ctx->stream);
  PL_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  const double warps = (double)blocks * threads / 32;
  const double flops = 2.0 * 256 * 8 * (double)iters * warps;
  *h_tflops = flops / (ms * 1e-3) / 1e12;
  return PL_OK;
}

}  // extern "C"
