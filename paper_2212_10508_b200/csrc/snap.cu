// SNAP placeholder (replaced by the fp64 bispectrum kernels).
#include "pl_common.cuh"
namespace pl {
int snap_prepare(pl_pot* pot, const double* h_beta) { (void)pot; (void)h_beta; return fail(PL_EARG, "SNAP not built yet"); }
void snap_release(pl_pot* pot) { (void)pot; }
int compute_snap(pl_pot* pot, int64_t B, const double* q, double* energy, double* grad, double* virial) {
  (void)pot; (void)B; (void)q; (void)energy; (void)grad; (void)virial;
  return fail(PL_EARG, "SNAP not built yet");
}
}
