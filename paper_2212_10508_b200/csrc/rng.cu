// Counter-based Gaussian noise streams (restates rng.py:57-185 for the GPU).
//
// The reference stream for a seed is the first `count` variates of the
// infinite sequence of accepted Marsaglia-polar pairs, pair i built from the
// counter uniforms j = 2i, 2i+1.  That makes the stream a stream-compaction
// problem: pass 1 counts accepted pairs per chunk of candidate pairs, a scan
// turns counts into output offsets, pass 2 recomputes the chunk and scatters
// x*f, y*f to their ranks.  Every CTA works on a disjoint chunk, so one launch
// covers all rows (windows x replicas) and the chip is full even for a
// single 48M-variate stream (heavy config).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "pl_common.cuh"

namespace pl {
namespace {

constexpr int RNG_THREADS = 256;
constexpr int RNG_PER_THREAD = 4;
constexpr int RNG_CHUNK = RNG_THREADS * RNG_PER_THREAD;  // candidate pairs per CTA

__device__ __forceinline__ double uniform(uint64_t seed, uint64_t j) {
  // (mix(seed + (j+1)*GOLDEN) >> 11) * 2^-53  (rng.py:81-84), wrapping u64
  uint64_t z = mix64(seed + (j + 1ull) * GOLDEN);
  return (double)(z >> 11) * 0x1.0p-53;
}

struct PairEval {
  double x, y, s;
  bool ok;
};

__device__ __forceinline__ PairEval eval_pair(uint64_t seed, uint64_t pair) {
  PairEval e;
  double u1 = uniform(seed, 2ull * pair);
  double u2 = uniform(seed, 2ull * pair + 1ull);
  e.x = sub(mul(2.0, u1), 1.0);
  e.y = sub(mul(2.0, u2), 1.0);
  e.s = add(mul(e.x, e.x), mul(e.y, e.y));
  e.ok = (e.s > 0.0) && (e.s < 1.0);
  return e;
}

__global__ void k_derive_seeds(uint64_t master, int64_t n, uint64_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = mix64(master ^ ((uint64_t)(i + 1) * GOLDEN));  // rng.py:66
}

// pass 1: accepted pairs per chunk
__global__ void __launch_bounds__(RNG_THREADS)
k_polar_count(const uint64_t* __restrict__ seeds, int64_t n_chunks, int32_t* __restrict__ counts) {
  int64_t row = blockIdx.y;
  int64_t chunk = blockIdx.x;
  uint64_t seed = seeds[row];
  uint64_t p0 = (uint64_t)chunk * RNG_CHUNK + (uint64_t)threadIdx.x * RNG_PER_THREAD;
  int c = 0;
#pragma unroll
  for (int k = 0; k < RNG_PER_THREAD; ++k) c += eval_pair(seed, p0 + k).ok ? 1 : 0;
  typedef cub::BlockReduce<int, RNG_THREADS> R;
  __shared__ typename R::TempStorage tmp;
  int sum = R(tmp).Sum(c);
  if (threadIdx.x == 0) counts[row * n_chunks + chunk] = sum;
}

// exclusive scan of chunk counts per row; flags rows whose accepted total is short
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS)
k_polar_scan(int32_t* __restrict__ counts, int64_t n_chunks, int64_t pairs_needed,
             int32_t* __restrict__ short_flag) {
  int64_t row = blockIdx.x;
  int32_t* c = counts + row * n_chunks;
  int64_t per = (n_chunks + SCAN_THREADS - 1) / SCAN_THREADS;
  int64_t lo = threadIdx.x * per;
  int64_t hi = lo + per < n_chunks ? lo + per : n_chunks;
  long long local = 0;
  for (int64_t i = lo; i < hi; ++i) local += c[i];
  typedef cub::BlockScan<long long, SCAN_THREADS> S;
  __shared__ typename S::TempStorage tmp;
  long long excl, total;
  S(tmp).ExclusiveSum(local, excl, total);
  for (int64_t i = lo; i < hi; ++i) {
    long long v = c[i];
    // offsets beyond pairs_needed are clamped: those chunks write nothing
    c[i] = (int32_t)(excl < pairs_needed ? excl : pairs_needed);
    excl += v;
  }
  if (threadIdx.x == 0 && total < pairs_needed) atomicExch(short_flag, 1);
}

// pass 2: recompute and scatter accepted pairs to their rank
__global__ void __launch_bounds__(RNG_THREADS)
k_polar_write(const uint64_t* __restrict__ seeds, int64_t n_chunks,
              const int32_t* __restrict__ offsets, int64_t count, double* __restrict__ out) {
  int64_t row = blockIdx.y;
  int64_t chunk = blockIdx.x;
  int64_t base = offsets[row * n_chunks + chunk];
  int64_t pairs_needed = (count + 1) / 2;
  if (base >= pairs_needed) return;  // whole CTA: uniform branch
  uint64_t seed = seeds[row];
  uint64_t p0 = (uint64_t)chunk * RNG_CHUNK + (uint64_t)threadIdx.x * RNG_PER_THREAD;
  PairEval e[RNG_PER_THREAD];
  int c = 0;
#pragma unroll
  for (int k = 0; k < RNG_PER_THREAD; ++k) {
    e[k] = eval_pair(seed, p0 + k);
    c += e[k].ok ? 1 : 0;
  }
  typedef cub::BlockScan<int, RNG_THREADS> S;
  __shared__ typename S::TempStorage tmp;
  int excl;
  S(tmp).ExclusiveSum(c, excl);
  int64_t rank = base + excl;
  double* o = out + row * count;
#pragma unroll
  for (int k = 0; k < RNG_PER_THREAD; ++k) {
    if (!e[k].ok) continue;
    if (rank < pairs_needed) {
      // f = sqrt(-2 log(s) / s)  (rng.py:99, 135); log is the only op with
      // implementation freedom (<= 1 ulp), all others are IEEE-exact here.
      double f = __dsqrt_rn(dvd(mul(-2.0, log(e[k].s)), e[k].s));
      int64_t i0 = 2 * rank;
      o[i0] = mul(e[k].x, f);
      if (i0 + 1 < count) o[i0 + 1] = mul(e[k].y, f);
    }
    ++rank;
  }
}

}  // namespace

int derive_seeds(pl_ctx* ctx, uint64_t master, int64_t n, uint64_t* out) {
  if (n < 0) return fail(PL_EARG, "n_windows must be >= 0");
  if (n == 0) return PL_OK;
  int64_t blocks = (n + 255) / 256;
  k_derive_seeds<<<(unsigned)blocks, 256, 0, ctx->stream>>>(master, n, out);
  PL_CHECK_LAUNCH();
  return PL_OK;
}

int gaussian_streams(pl_ctx* ctx, const uint64_t* seeds, int64_t n_rows, int64_t count,
                     double* out) {
  if (n_rows < 0 || count < 0) return fail(PL_EARG, "n_rows and count must be >= 0");
  if (n_rows == 0 || count == 0) return PL_OK;
  if (n_rows > 65535) return fail(PL_EARG, "at most 65535 rows per call");
  int64_t pairs = (count + 1) / 2;
  // acceptance pi/4: expected 1.273*pairs candidates; +10 sigma + slack
  double sd = sqrt((double)pairs);
  int64_t cand = (int64_t)(1.2733 * (double)pairs + 10.0 * sd + 64.0);
  for (int attempt = 0; attempt < 8; ++attempt) {
    int64_t n_chunks = (cand + RNG_CHUNK - 1) / RNG_CHUNK;
    if (n_chunks > 0x7fffffff) return fail(PL_EARG, "noise stream too long");
    size_t need = (size_t)n_rows * n_chunks * sizeof(int32_t) + 256;
    PL_TRY(ctx->work[0].reserve(need));
    int32_t* counts = (int32_t*)ctx->work[0].ptr;
    int32_t* flag = (int32_t*)((char*)ctx->work[0].ptr + (size_t)n_rows * n_chunks * 4);
    flag = (int32_t*)(((uintptr_t)flag + 15) & ~(uintptr_t)15);
    PL_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), ctx->stream));
    dim3 grid((unsigned)n_chunks, (unsigned)n_rows);
    k_polar_count<<<grid, RNG_THREADS, 0, ctx->stream>>>(seeds, n_chunks, counts);
    PL_CHECK_LAUNCH();
    k_polar_scan<<<(unsigned)n_rows, SCAN_THREADS, 0, ctx->stream>>>(counts, n_chunks, pairs, flag);
    PL_CHECK_LAUNCH();
    int32_t h_flag = 0;
    PL_CUDA(cudaMemcpyAsync(&h_flag, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    PL_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!h_flag) {
      k_polar_write<<<grid, RNG_THREADS, 0, ctx->stream>>>(seeds, n_chunks, counts, count, out);
      PL_CHECK_LAUNCH();
      return PL_OK;
    }
    cand *= 2;
  }
  return fail(PL_EARG, "polar stream acceptance shortfall");
}

}  // namespace pl
