// extern "C" surface of paralangevin_b200 (declared in include/paralangevin_b200.h).
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "neigh.cuh"
#include "pl_common.cuh"

namespace pl {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int Scratch::reserve(size_t n) {
  if (n <= bytes) return PL_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
  size_t want = n + n / 4 + 256;
  cudaError_t e = cudaMalloc(&ptr, want);
  if (e != cudaSuccess) return fail(PL_ECUDA, std::string("cudaMalloc scratch: ") + cudaGetErrorString(e));
  bytes = want;
  return PL_OK;
}
Scratch::~Scratch() {
  if (ptr) cudaFree(ptr);
}

int derive_seeds(pl_ctx* ctx, uint64_t master, int64_t n, uint64_t* out);
int gaussian_streams(pl_ctx* ctx, const uint64_t* seeds, int64_t n_rows, int64_t count, double* out);
int propagate_windows(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L, const double* q0,
                      const double* p0, const double* noise, const double* h_amp,
                      const double* mass, double dt, double h, double hg, double* q1, double* p1,
                      int32_t* blow, double* s1 = nullptr, double* s2 = nullptr);
int lj_check(pl_pot* pot);
int minimize(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, double* x, double tol, int64_t max_iter,
             int32_t* h_status, int64_t* h_iters, double* h_energy);
int eam_prepare(pl_pot* pot, const double* rho, const double* phi, const double* F);
int sweep(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int include_m0,
          double* traj_q, double* traj_p, const double* prev_q, double* base_q, double* base_p,
          const double* jump_q, const double* jump_p, const double* noise_all, const double* h_amp,
          const double* mass, double dt, double h, double hg, double expl, double* h_state,
          double* d_hist, int64_t* h_out, int32_t* h_blowup);

static int upload(pl_ctx* ctx, const double* h, int64_t n, double** d) {
  *d = nullptr;
  if (!h || n <= 0) return PL_OK;
  PL_CUDA(cudaMalloc(d, sizeof(double) * n));
  PL_CUDA(cudaMemcpy(*d, h, sizeof(double) * n, cudaMemcpyHostToDevice));
  (void)ctx;
  return PL_OK;
}

static bool finite_all(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

}  // namespace pl

using namespace pl;

extern "C" {

int pl_version(void) { return 100; }
const char* pl_last_error(void) { return g_err.c_str(); }

int pl_ctx_create(int device, void* stream, pl_ctx** out) {
  if (!out) return fail(PL_EARG, "out is NULL");
  PL_CUDA(cudaSetDevice(device));
  pl_ctx* c = new pl_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  *out = c;
  return PL_OK;
}

int pl_ctx_set_stream(pl_ctx* ctx, void* stream) {
  if (!ctx) return fail(PL_EARG, "ctx is NULL");
  ctx->stream = (cudaStream_t)stream;
  return PL_OK;
}

int pl_ctx_enable_progress(pl_ctx* ctx, int64_t** h_progress) {
  if (!ctx || !h_progress) return fail(PL_EARG, "NULL argument");
  if (!ctx->progress) {
    void* p = nullptr;
    PL_CUDA(cudaHostAlloc(&p, 64, cudaHostAllocMapped));
    void* dp = nullptr;
    PL_CUDA(cudaHostGetDevicePointer(&dp, p, 0));
    ctx->progress = (int64_t*)p;
    ctx->progress_dev = (int64_t*)dp;
    *(volatile int64_t*)ctx->progress = 0;
  }
  *h_progress = ctx->progress;
  return PL_OK;
}

int pl_ctx_set_spec(pl_ctx* ctx, int on) {
  if (!ctx) return fail(PL_EARG, "ctx is NULL");
  ctx->spec = on ? 1 : 0;
  return PL_OK;
}

int pl_ctx_synchronize(pl_ctx* ctx) {
  if (!ctx) return fail(PL_EARG, "ctx is NULL");
  PL_CUDA(cudaStreamSynchronize(ctx->stream));
  return PL_OK;
}

int pl_ctx_destroy(pl_ctx* ctx) {
  if (!ctx) return PL_OK;
  cudaStreamSynchronize(ctx->stream);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->progress) cudaFreeHost(ctx->progress);
  delete ctx;
  return PL_OK;
}

int pl_derive_seeds(pl_ctx* ctx, uint64_t master, int64_t n, uint64_t* d_out) {
  if (!ctx) return fail(PL_EARG, "ctx is NULL");
  return derive_seeds(ctx, master, n, d_out);
}

int pl_gaussian_streams(pl_ctx* ctx, const uint64_t* d_seeds, int64_t n_rows, int64_t count,
                        double* d_out) {
  if (!ctx) return fail(PL_EARG, "ctx is NULL");
  return gaussian_streams(ctx, d_seeds, n_rows, count, d_out);
}

static pl_pot* new_pot(pl_ctx* ctx, PotKind k) {
  pl_pot* p = new pl_pot();
  p->ctx = ctx;
  p->kind = k;
  return p;
}

int pl_pot_free(pl_ctx* ctx, pl_pot** out) {
  if (!ctx || !out) return fail(PL_EARG, "NULL argument");
  *out = new_pot(ctx, POT_FREE);
  return PL_OK;
}

static int coeff_pot(pl_ctx* ctx, PotKind k, int64_t dim, const double* a, const double* b,
                     pl_pot** out) {
  if (!ctx || !out || !a) return fail(PL_EARG, "NULL argument");
  if (dim < 0) return fail(PL_EARG, "dim must be >= 0");
  int64_t n = dim ? dim : 1;
  if (!finite_all(a, n) || (b && !finite_all(b, n))) return fail(PL_EARG, "coefficients must be finite");
  for (int64_t i = 0; i < n; ++i)
    if (!(a[i] > 0.0) || (b && !(b[i] > 0.0))) return fail(PL_EARG, "coefficients must be positive");
  pl_pot* p = new_pot(ctx, k);
  p->dim = dim;
  if (dim == 0) {
    p->s0 = a[0];
    p->s1 = b ? b[0] : 0.0;
  } else {
    int rc = upload(ctx, a, dim, &p->d_c0);
    if (rc == PL_OK && b) rc = upload(ctx, b, dim, &p->d_c1);
    if (rc != PL_OK) {
      delete p;
      return rc;
    }
  }
  *out = p;
  return PL_OK;
}

int pl_pot_harmonic(pl_ctx* ctx, int64_t dim, const double* h_k, pl_pot** out) {
  return coeff_pot(ctx, POT_HARMONIC, dim, h_k, nullptr, out);
}

int pl_pot_double_well(pl_ctx* ctx, int64_t dim, const double* h_a, const double* h_b, pl_pot** out) {
  if (!h_b) return fail(PL_EARG, "b is NULL");
  return coeff_pot(ctx, POT_DOUBLE_WELL, dim, h_a, h_b, out);
}

int pl_pot_lj(pl_ctx* ctx, double eps, double sigma, int n_atoms, int space_dim, pl_pot** out) {
  if (!ctx || !out) return fail(PL_EARG, "NULL argument");
  if (!(std::isfinite(eps) && eps > 0.0)) return fail(PL_EARG, "epsilon must be positive");
  if (!(std::isfinite(sigma) && sigma > 0.0)) return fail(PL_EARG, "sigma must be positive");
  if (n_atoms < 2) return fail(PL_EARG, "need at least 2 atoms");
  if (space_dim < 1 || space_dim > 3) return fail(PL_EARG, "space_dim must be 1..3 on the device");
  pl_pot* p = new_pot(ctx, POT_LJ);
  p->eps = eps;
  p->sigma = sigma;
  p->n_atoms = n_atoms;
  p->space_dim = space_dim;
  p->dim = (int64_t)n_atoms * space_dim;
  *out = p;
  return PL_OK;
}

int pl_pot_perturbed(pl_ctx* ctx, pl_pot* base, pl_pot* delta, double lam, pl_pot** out) {
  if (!ctx || !base || !delta || !out) return fail(PL_EARG, "NULL argument");
  if (!std::isfinite(lam)) return fail(PL_EARG, "lam must be finite");
  if (base->dim && delta->dim && base->dim != delta->dim)
    return fail(PL_EARG, "base and delta have incompatible dimensions");
  pl_pot* p = new_pot(ctx, POT_PERTURBED);
  p->base = base;
  p->delta = delta;
  p->lam = lam;
  p->dim = base->dim ? base->dim : delta->dim;
  p->flops = base->flops + (lam != 0.0 ? delta->flops : 0.0);
  *out = p;
  return PL_OK;
}

static int check_box(const double* box, double rcut, int n_atoms) {
  if (!box) return fail(PL_EARG, "box is NULL");
  if (n_atoms < 1) return fail(PL_EARG, "n_atoms must be >= 1");
  for (int c = 0; c < 3; ++c) {
    if (!(std::isfinite(box[c]) && box[c] > 0.0)) return fail(PL_EARG, "box lengths must be positive");
    // single-image minimum convention: every pair within rcut is unique
    if (box[c] < 2.0 * rcut) return fail(PL_EPOT, "box length below 2*rcut (minimum image not unique)");
  }
  return PL_OK;
}

int pl_pot_eam(pl_ctx* ctx, int n_atoms, const double* h_box, double rcut, int n_r, double dr,
               const double* h_rho, const double* h_phi, int n_rho, double drho, const double* h_F,
               pl_pot** out) {
  if (!ctx || !out || !h_rho || !h_phi || !h_F) return fail(PL_EARG, "NULL argument");
  PL_TRY(check_box(h_box, rcut, n_atoms));
  if (n_r < 2 || n_rho < 2 || !(dr > 0) || !(drho > 0)) return fail(PL_EARG, "bad EAM table");
  pl_pot* p = new_pot(ctx, POT_EAM);
  p->n_atoms = n_atoms;
  p->dim = 3 * (int64_t)n_atoms;
  std::memcpy(p->box, h_box, sizeof(double) * 3);
  p->rcut = rcut;
  p->n_r = n_r;
  p->dr = dr;
  p->n_rho = n_rho;
  p->drho = drho;
  int rc = eam_prepare(p, h_rho, h_phi, h_F);
  if (rc != PL_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return PL_OK;
}

int pl_pot_snap(pl_ctx* ctx, int n_atoms, const double* h_box, int twojmax, double rcut,
                double rfac0, double rmin0, int switchflag, double wself, const double* h_beta,
                int nbeta, pl_pot** out) {
  if (!ctx || !out || !h_beta) return fail(PL_EARG, "NULL argument");
  PL_TRY(check_box(h_box, rcut, n_atoms));
  if (twojmax < 0 || twojmax > 14) return fail(PL_EARG, "twojmax must be in 0..14");
  if (!(rfac0 > 0.0 && rfac0 < 1.0)) return fail(PL_EARG, "rfac0 must lie in (0, 1)");
  if (!(rmin0 >= 0.0 && rmin0 < rcut)) return fail(PL_EARG, "rmin0 must lie in [0, rcut)");
  pl_pot* p = new_pot(ctx, POT_SNAP);
  p->n_atoms = n_atoms;
  p->dim = 3 * (int64_t)n_atoms;
  std::memcpy(p->box, h_box, sizeof(double) * 3);
  p->rcut = rcut;
  p->twojmax = twojmax;
  p->rfac0 = rfac0;
  p->rmin0 = rmin0;
  p->switchflag = switchflag;
  p->wself = wself;
  p->nbeta = nbeta;
  // Verlet skin of the in-window lists (PL_SNAP_SKIN, A; 0 = exact lists every substep):
  // 0.3 A keeps the BCC W lists below the fourth shell (5.25 A) at rcut 4.73 A
  {
    const char* e = std::getenv("PL_SNAP_SKIN");
    p->skin = e ? std::atof(e) : 0.3;
    if (!(p->skin >= 0.0 && p->skin < rcut)) p->skin = 0.0;
  }
  int rc = snap_prepare(p, h_beta);
  if (rc != PL_OK) {
    delete p;
    return rc;
  }
  *out = p;
  return PL_OK;
}

int pl_pot_destroy(pl_pot* p) {
  // does not touch p->ctx: contexts and potentials may be released in any order
  // (e.g. at interpreter shutdown); cudaFree synchronises with the device itself
  if (!p) return PL_OK;
  cudaFree(p->d_c0);
  cudaFree(p->d_c1);
  cudaFree(p->d_rho);
  cudaFree(p->d_phi);
  cudaFree(p->d_F);
  if (p->kind == POT_SNAP) snap_release(p);
  delete p;
  return PL_OK;
}

double pl_pot_flops(pl_pot* p) { return p ? p->flops : 0.0; }

int pl_compute(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, const double* d_q, double* d_energy,
               double* d_grad, double* d_virial) {
  if (!ctx || !pot || !d_q) return fail(PL_EARG, "NULL argument");
  if (B < 0 || d < 1) return fail(PL_EARG, "need B >= 0 and d >= 1");
  PL_TRY(compute(pot, B, d, d_q, d_energy, d_grad, d_virial));
  if (pot->kind == POT_LJ) return lj_check(pot);
  return neigh_check(pot);
}

int pl_neighbours(pl_ctx* ctx, pl_pot* pot, int64_t B, const double* d_q, int maxn, int32_t* d_nbr,
                  int32_t* d_cnt) {
  if (!ctx || !pot || !d_q || !d_nbr || !d_cnt) return fail(PL_EARG, "NULL argument");
  if (pot->kind != POT_EAM && pot->kind != POT_SNAP) return fail(PL_EARG, "not a periodic potential");
  if (maxn < 1) return fail(PL_EARG, "maxn must be >= 1");
  NeighList nl;
  PL_TRY(build_neighbours(pot, B, d_q, pot->rcut, maxn, &nl));
  PL_CUDA(cudaMemcpyAsync(d_nbr, nl.nbr, sizeof(int32_t) * B * pot->n_atoms * maxn,
                          cudaMemcpyDeviceToDevice, ctx->stream));
  PL_CUDA(cudaMemcpyAsync(d_cnt, nl.cnt, sizeof(int32_t) * B * pot->n_atoms, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  return neigh_check(pot);
}

int pl_propagate_windows(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L,
                         const double* d_q0, const double* d_p0, const double* d_noise,
                         const double* h_amp, const double* d_mass, double dt, double half_dt,
                         double half_dt_gamma, double* d_q1, double* d_p1, int32_t* d_blowup) {
  if (!ctx || !pot || !d_q0 || !d_p0 || !d_noise || !h_amp || !d_q1 || !d_p1 || !d_blowup)
    return fail(PL_EARG, "NULL argument");
  return propagate_windows(ctx, pot, W, d, L, d_q0, d_p0, d_noise, h_amp, d_mass, dt, half_dt,
                           half_dt_gamma, d_q1, d_p1, d_blowup);
}

int pl_minimize(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, double* d_x, double tol, int64_t max_iter,
                int32_t* h_status, int64_t* h_iters, double* h_energy) {
  if (!ctx || !pot || !d_x || !h_status || !h_iters) return fail(PL_EARG, "NULL argument");
  return minimize(ctx, pot, B, d, d_x, tol, max_iter, h_status, h_iters, h_energy);
}

int pl_propagate_windows_moments(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L,
                                 const double* d_q0, const double* d_p0, const double* d_noise,
                                 const double* h_amp, const double* d_mass, double dt, double half_dt,
                                 double half_dt_gamma, double* d_q1, double* d_p1, int32_t* d_blowup,
                                 double* d_s1, double* d_s2) {
  if (!ctx || !pot || !d_q0 || !d_p0 || !d_noise || !h_amp || !d_q1 || !d_p1 || !d_blowup || !d_s1 || !d_s2)
    return fail(PL_EARG, "NULL argument");
  return propagate_windows(ctx, pot, W, d, L, d_q0, d_p0, d_noise, h_amp, d_mass, dt, half_dt, half_dt_gamma,
                           d_q1, d_p1, d_blowup, d_s1, d_s2);
}

int pl_sweep(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1, int include_m0,
             double* d_traj_q, double* d_traj_p, const double* d_prev_q, double* d_base_q,
             double* d_base_p, const double* d_jump_q, const double* d_jump_p,
             const double* d_noise_all, const double* h_amp, const double* d_mass, double dt,
             double half_dt, double half_dt_gamma, double expl, double* h_state, double* d_hist,
             int64_t* h_out, int32_t* h_blowup) {
  if (!ctx || !coarse || !d_traj_q || !d_traj_p || !d_prev_q || !d_base_q || !d_base_p ||
      !d_jump_q || !d_jump_p || !d_noise_all || !h_amp || !h_state || !d_hist || !h_out || !h_blowup)
    return fail(PL_EARG, "NULL argument");
  if (d < 1 || L < 1 || m0 < 0) return fail(PL_EARG, "need d >= 1, L >= 1, m0 >= 0");
  return sweep(ctx, coarse, d, L, m0, m1, include_m0, d_traj_q, d_traj_p, d_prev_q, d_base_q,
               d_base_p, d_jump_q, d_jump_p, d_noise_all, h_amp, d_mass, dt, half_dt,
               half_dt_gamma, expl, h_state, d_hist, h_out, h_blowup);
}

}  // extern "C"
