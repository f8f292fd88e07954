// Shared internals of the paralangevin_b200 C ABI (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "paralangevin_b200.h"

namespace pl {

// ---- error reporting (thread-local, no global mutable state shared across threads)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

// Device-side bounds checks (build.py --variant checks -DPL_CHECKS): the index
// and capacity invariants of the hot kernels, trapping on violation.  The
// compute-sanitizer stand-in on a pool where it is closed.
#ifdef PL_CHECKS
#include <cassert>
#define PL_DASSERT(cond) assert(cond)
#else
#define PL_DASSERT(cond) ((void)0)
#endif

#define PL_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return ::pl::fail(PL_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define PL_CHECK_LAUNCH() PL_CUDA(cudaGetLastError())

#define PL_TRY(call)              \
  do {                            \
    int _rc = (call);             \
    if (_rc != PL_OK) return _rc; \
  } while (0)

// ---- programmatic dependent launch: the kernels of one force evaluation and
// the integrator steps around it are launched with programmatic stream
// serialisation, so a grid's launch is processed while its predecessor runs;
// every such kernel waits for the predecessor's completion (griddep_wait) before
// it touches memory, so the ordering is the stream's.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- once-per-device setup (function attributes, __constant__ tables): true
// the first time it is called on the current device for this mask.  Device
// state is per device, so a process-wide flag would skip a second GPU.
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = 1ull << dev;
  return (mask.fetch_or(bit) & bit) == 0;
}

// ---- exact-order fp64 arithmetic: no FMA contraction on the parity path.
// numpy evaluates left to right with one rounding per operation
// (integrator.py:174-177, rng.py:130-135); these intrinsics pin that.
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dvd(double a, double b) { return __ddiv_rn(a, b); }

// ---- SplitMix64 (rng.py:31-45)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;
constexpr double BLOWUP_LIMIT = 1e12;

// ---- device workspace: grow-only scratch owned by a context
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  int reserve(size_t n);
  ~Scratch();
};

}  // namespace pl

// Potential kinds
enum PotKind {
  POT_FREE = 0,
  POT_HARMONIC = 1,
  POT_DOUBLE_WELL = 2,
  POT_LJ = 3,
  POT_PERTURBED = 4,
  POT_EAM = 5,
  POT_SNAP = 6,
};

namespace pl { struct SnapIndex; }  // snap.cu

struct pl_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  pl::Scratch work[10];  // named slots, see pl_ctx slot enum in each .cu (8, 9: speculative windows)
  // speculative mode (pl_ctx_set_spec): window propagation defers its neighbour-
  // capacity check (no host synchronisation; pl_pot_overflow_async reads the flag
  // on the stream) and uses its own integrator scratch slots, so it can run on a
  // second stream next to a sweep on the first
  int spec = 0;
  // host-mapped progress counter (pl_ctx_enable_progress): the single-replica
  // cluster sweep stores the number of windows it has finished after each one
  int64_t* progress = nullptr;      // host pointer
  int64_t* progress_dev = nullptr;  // its device alias
  // pinned host staging for small scalars read back by sync calls
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
};

struct pl_pot {
  pl_ctx* ctx = nullptr;
  PotKind kind = POT_FREE;
  int64_t dim = 0;  // fixed dimension, 0 = any
  // elementwise coefficients (device): harmonic k / double-well a, b
  double* d_c0 = nullptr;
  double* d_c1 = nullptr;
  double s0 = 0.0, s1 = 0.0;  // scalar coefficients when dim == 0
  // LJ
  double eps = 1.0, sigma = 1.0;
  int n_atoms = 0, space_dim = 0;
  // perturbed
  pl_pot* base = nullptr;
  pl_pot* delta = nullptr;
  double lam = 0.0;
  // periodic many-body potentials
  double box[3] = {0, 0, 0};
  double rcut = 0.0;
  // EAM tables (device)
  int n_r = 0, n_rho = 0;
  double dr = 0.0, drho = 0.0;
  double* d_rho = nullptr;
  double* d_phi = nullptr;
  double* d_F = nullptr;
  // SNAP
  int twojmax = 0;
  double rfac0 = 0.0, rmin0 = 0.0, wself = 1.0;
  int switchflag = 1;
  int nbeta = 0;
  pl::SnapIndex* snap = nullptr;
  double flops = 0.0;
  int* nb_overflow = nullptr;  // device flag: neighbour capacity exceeded since the last check (sticky)
  bool nb_armed = true;        // the next neighbour build clears the flag (set by every check)
  // Verlet skin of the SNAP lists inside a window propagation (snap.cu): lists to
  // rcut + skin, rebuilt on the device only when an atom moved more than skin/2
  // since the last build; every SNAP kernel compacts the exact pairs (r < rcut)
  // in list order, so the forces are bitwise those of exact lists
  double skin = 0.0;
  bool skin_on = false;     // set by propagate_windows for its duration
  bool skin_force = false;  // next evaluation rebuilds unconditionally (window start)
  int64_t skin_B = -1;      // batch size of the current skin lists
  // per-potential scratch (neighbour lists, per-atom buffers)
  pl::Scratch work[8];
};

namespace pl {
bool is_elementwise(const pl_pot* p);
// Generic batched gradient (+energy) of B systems of dimension d on ctx->stream.
int compute(pl_pot* pot, int64_t B, int64_t d, const double* q, double* energy, double* grad,
            double* virial);
int compute_eam(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad,
                double* virial);
int compute_snap(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad,
                 double* virial);
int snap_prepare(pl_pot* pot, const double* h_beta);
int neigh_check(pl_pot* pot);
// live stage timing (prof.cu): stages 0 neigh, 1 snap_ui, 2 snap_yi, 3 snap_deidrj,
// 4 snap_gather, 5 eam, 6 integrator
enum ProfStage { ST_NEIGH = 0, ST_UI = 1, ST_YI = 2, ST_DE = 3, ST_GATHER = 4, ST_EAM = 5, ST_INT = 6 };
void prof_mark(cudaStream_t st, int stage, bool begin);
void snap_release(pl_pot* pot);
}  // namespace pl
