/*
 * paralangevin_b200 -- C ABI of the B200-native parareal / SNAP hot path.
 *
 * The reference (arXiv 2212.10508 package `paralangevin`, pure Python) has no
 * FFI; its plug-in boundaries are Python protocols.  Each entry point below
 * replaces one of them, batched over many windows/systems:
 *
 *   pl_derive_seeds        rng.py:69-78        derive_seeds(master, n)
 *   pl_gaussian_streams    rng.py:154-185      gaussian_stream(s)(seed, count)
 *   pl_pot_*               potentials.py:62-214 Potential subclasses (+ EAM, SNAP)
 *   pl_compute             potentials.py:45-49 Potential.energy / .gradient
 *   pl_propagate_windows   integrator.py:259-308 propagate_window (W windows)
 *   pl_sweep               parareal.py:289-299, 195-198, 425-445
 *                          corrected coarse sweep + running relative error
 *
 * Conventions
 *   - every array argument prefixed d_ is a DEVICE pointer (cudaMalloc /
 *     torch CUDA tensor); h_ is host memory.  No torch types cross the ABI.
 *   - states are the reference's flat atom-major fp64 vectors
 *     q = (x0, y0, z0, x1, ...) (potentials.py:135-136); a batch of W states
 *     is W consecutive vectors of length d.
 *   - calls are asynchronous on the context's stream unless noted; all
 *     return an int status (PL_OK, ...).  pl_last_error() gives the message.
 *   - no global mutable state: a context may be used by one host thread at a
 *     time; distinct contexts are independent (thread-safe).
 */
#ifndef PARALANGEVIN_B200_H
#define PARALANGEVIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PL_OK = 0,
  PL_EARG = 2,      /* bad argument (ValueError / PotentialError)            */
  PL_EBLOWUP = 3,   /* a window left |x| <= 1e12 (integrator.py:163-170)     */
  PL_EPOT = 4,      /* potential cannot evaluate (e.g. box too small, r = 0) */
  PL_ECUDA = 5      /* CUDA runtime error                                    */
};

typedef struct pl_ctx pl_ctx;
typedef struct pl_pot pl_pot;

int pl_version(void);
const char* pl_last_error(void);

/* Context: device + stream (cudaStream_t passed as void*; NULL = legacy). */
int pl_ctx_create(int device, void* stream, pl_ctx** out);
int pl_ctx_set_stream(pl_ctx* ctx, void* stream);
/* Speculative mode (on != 0): window propagation does not synchronise the host
 * for its neighbour-capacity check (read it later with pl_pot_overflow_async)
 * and uses its own scratch, so speculative fine windows can be launched on a
 * second stream while a corrected sweep runs on the first (parareal.py
 * pipelining; no reference counterpart). */
int pl_ctx_set_spec(pl_ctx* ctx, int on);
/* Host-mapped progress counter of this context: single-replica cluster sweeps
 * store the number of windows finished after each window (read it while the
 * blocking pl_sweep runs in another host thread).  *h_progress = its address. */
int pl_ctx_enable_progress(pl_ctx* ctx, int64_t** h_progress);
/* 2 if a single-replica sweep with this coarse potential runs as the persistent
 * cluster kernel (the one that reports progress), 0 otherwise; < 0 on error. */
int pl_sweep_path(pl_pot* coarse);
int pl_ctx_synchronize(pl_ctx* ctx);
int pl_ctx_destroy(pl_ctx* ctx);

/* ---- noise (rng.py) ---------------------------------------------------- */
/* d_out[n-1] = derive_seed(master, n), n = 1..n_windows  (rng.py:57-78). */
int pl_derive_seeds(pl_ctx* ctx, uint64_t master, int64_t n_windows, uint64_t* d_out);
/* Row r of d_out (n_rows x count) = gaussian_stream(d_seeds[r], count)
 * (rng.py:87-185): SplitMix64 counter uniforms, Marsaglia polar with
 * rejection, accepted pairs in counter order.  Bit-exact except for the
 * 1-ulp freedom of log(); see DESIGN.md.  Synchronises (acceptance check). */
int pl_gaussian_streams(pl_ctx* ctx, const uint64_t* d_seeds, int64_t n_rows, int64_t count,
                        double* d_out);

/* ---- potentials (potentials.py) ---------------------------------------- */
/* dim = 0 means "scalar coefficient, any dimension" (potentials.py:25-36). */
int pl_pot_free(pl_ctx* ctx, pl_pot** out);
int pl_pot_harmonic(pl_ctx* ctx, int64_t dim, const double* h_k, pl_pot** out);
int pl_pot_double_well(pl_ctx* ctx, int64_t dim, const double* h_a, const double* h_b,
                       pl_pot** out);
int pl_pot_lj(pl_ctx* ctx, double epsilon, double sigma, int n_atoms, int space_dim,
              pl_pot** out);
/* V = base + lam * delta; lam == 0 returns base bit for bit (potentials.py:183-214).
 * The new handle references (does not own) base and delta. */
int pl_pot_perturbed(pl_ctx* ctx, pl_pot* base, pl_pot* delta, double lam, pl_pot** out);
/* Tabulated EAM (Finnis-Sinclair form E = sum_i F(rho_i) + 1/2 sum phi(r_ij)).
 * rho(r), phi(r): n_r cubic pieces on [0, rcut] (coef layout [n_r][4],
 * value = c0 + t(c1 + t(c2 + t c3)), t = r/dr - k).  F(rho): n_rho pieces
 * on [0, n_rho*drho].  Orthorhombic periodic box (box[3], Angstrom). */
int pl_pot_eam(pl_ctx* ctx, int n_atoms, const double* h_box, double rcut, int n_r, double dr,
               const double* h_rho_coef, const double* h_phi_coef, int n_rho, double drho,
               const double* h_F_coef, pl_pot** out);
/* SNAP (single element): E_i = beta[0] + sum_k beta[k] B_k(i), B over the
 * canonical (j1 >= j2, j >= j1) triples, U_tot with self weight wself,
 * cosine switch (switchflag = 1) on [rmin0, rcut]. nbeta = 1 + n_B(twojmax). */
int pl_pot_snap(pl_ctx* ctx, int n_atoms, const double* h_box, int twojmax, double rcut,
                double rfac0, double rmin0, int switchflag, double wself, const double* h_beta,
                int nbeta, pl_pot** out);
int pl_pot_destroy(pl_pot* pot);
/* SNAP per-atom bispectrum components B (B*n_atoms x n_B), canonical order
 * (j1 ascending, j2 <= j1 ascending, J ascending).  Parity/debug path. */
int pl_snap_bispectrum(pl_ctx* ctx, pl_pot* pot, int64_t B, const double* d_q, double* d_out);
/* SNAP index sizes {nhalf, nfull, n_B, n_items, n_units} and the algorithmic
 * fp64 FLOP counts {per pair (U), per atom (Z/Y), per pair (dU + contraction)}. */
int pl_snap_info(pl_pot* pot, int32_t* h_counts, double* h_flops);
/* Expected fp64 FLOPs of one evaluation of one system (algorithmic count). */
double pl_pot_flops(pl_pot* pot);

/* Full periodic neighbour lists the potential builds (ascending j, minimum
 * image, r^2 < rcut^2 with exact rounding): d_nbr (B*n_atoms*maxn), d_cnt
 * (B*n_atoms).  Returns PL_EPOT if a list exceeds maxn.  Synchronises. */
int pl_neighbours(pl_ctx* ctx, pl_pot* pot, int64_t B, const double* d_q, int maxn,
                  int32_t* d_nbr, int32_t* d_cnt);

/* ---- batched Potential.energy / gradient -------------------------------- */
/* B systems of dimension d: d_q (B*d); outputs may be NULL.
 * d_energy (B), d_grad (B*d), d_virial (B*6: xx yy zz xy xz yz). */
int pl_compute(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, const double* d_q,
               double* d_energy, double* d_grad, double* d_virial);

/* ---- batched window propagation (integrator.py:259-308) ---------------- */
/* W windows of L substeps.  d_noise: W x (L+1) x d Gaussian blocks (block l
 * of window w at d_noise[(w*(L+1)+l)*d]); h_amp: L+1 scalar amplitudes
 * 0.5*sqrt(2*gamma*C_l*inv_beta*dt) (integrator.py:156-160); d_mass: d masses
 * or NULL for unit mass.  half_dt = 0.5*dt and half_dt_gamma = 0.5*dt*gamma as
 * Python evaluates them.  d_blowup[w] = first substep (1-based) at which the
 * window left the trusted range, 0 if none.  Inputs are never modified;
 * outputs may alias inputs (in-place). */
int pl_propagate_windows(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L,
                         const double* d_q0, const double* d_p0, const double* d_noise,
                         const double* h_amp, const double* d_mass, double dt, double half_dt,
                         double half_dt_gamma, double* d_q1, double* d_p1, int32_t* d_blowup);

/* Same propagation, also accumulating the full-step momentum moments of the
 * kinetic-temperature measurement (integrator.py:350-365 _measure_chain,
 * 430-482 measure_kinetic_temperature): for every window w, substep
 * l = 1..L and component c,
 *   d_s1[(w*L + l-1)*d + c] += p_l,   d_s2[...] += p_l * p_l   (numpy order).
 * d_s1 / d_s2 are W x L x d device arrays owned by the caller (zero them
 * before the first window that counts). */
int pl_propagate_windows_moments(pl_ctx* ctx, pl_pot* pot, int64_t W, int64_t d, int L,
                                 const double* d_q0, const double* d_p0, const double* d_noise,
                                 const double* h_amp, const double* d_mass, double dt, double half_dt,
                                 double half_dt_gamma, double* d_q1, double* d_p1, int32_t* d_blowup,
                                 double* d_s1, double* d_s2);

/* ---- batched local minimisation (potentials.py:231-287) ---------------- */
/* B independent steepest descents with Armijo backtracking, the reference's
 * _descend: from x (B x d, device, overwritten with the result) until
 * sqrt(|grad|^2) <= tol, the step doubling (cap 1e3) per iteration and halving
 * per rejected trial, acceptance E_trial <= E - 0.5*step*|grad|^2 (a trial the
 * potential rejects counts as +inf).  h_status[b]: 0 converged, 1 line search
 * stalled (step < 1e-18), 2 no convergence within max_iter (the two cases
 * where the reference raises MinimizationError); h_iters[b] = accepted steps;
 * h_energy (optional) = final energies.  Synchronous. */
int pl_minimize(pl_ctx* ctx, pl_pot* pot, int64_t B, int64_t d, double* d_x, double tol, int64_t max_iter,
                int32_t* h_status, int64_t* h_iters, double* h_energy);

/* ---- parareal corrected sweep (parareal.py:289-299, 195-198, 425-445) -- */
/* Trajectory nodes live in two (N+1) x d arrays: d_traj_q, d_traj_p.  Window
 * quantities (indexed by the absolute 0-based window m) live in N x d arrays:
 * d_base_* (coarse(cur[m]), the cached C(prev[m]) of the next iteration --
 * SURVEY.md finding 7) and d_jump_* (F(prev[m]) - C(prev[m])).  For
 * m = m0 .. m1-1, sequentially:
 *   base[m] = coarse(cur[m]);  cur[m+1] = base[m] + jump[m];
 *   num += ||cur[m+1].q - prev[m+1].q||_2;  den += ||prev[m+1].q||_2
 *   hist[m - m0] = num / den
 * include_m0 != 0 first accumulates node m0 (parareal.py:423-424).  If
 * expl > 0 the sweep stops after the first node whose running error exceeds
 * expl (parareal.py:435-445).  h_state in/out {num, den}; h_out[0] = nodes
 * updated.  On a coarse blow-up returns PL_EBLOWUP with h_out[0] = window m,
 * h_blowup[0] = substep; a non-finite corrected state returns PL_EBLOWUP with
 * h_blowup[0] = 0.  d_noise_all: N x (L+1) x d.  EAM and elementwise coarse
 * potentials run the whole sweep in one persistent CTA (sweep_cta.cu); others
 * loop over windows on the host.  Synchronises. */
int pl_sweep(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1,
             int include_m0, double* d_traj_q, double* d_traj_p, const double* d_prev_q,
             double* d_base_q, double* d_base_p, const double* d_jump_q,
             const double* d_jump_p, const double* d_noise_all, const double* h_amp,
             const double* d_mass, double dt, double half_dt, double half_dt_gamma,
             double expl, double* h_state, double* d_hist, int64_t* h_out,
             int32_t* h_blowup);

/* Coarse bootstrap of a new slab (parareal.py:404-405): for m = m0..m1-1,
 * base[m] = coarse(cur[m]) and cur[m+1] = base[m] exactly.  On a blow-up
 * returns PL_EBLOWUP with h_out[0] = window m and h_blowup[0] = substep;
 * otherwise h_out[0] = windows done.  Synchronises. */
int pl_bootstrap(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t m0, int64_t m1,
                 double* d_traj_q, double* d_traj_p, double* d_base_q, double* d_base_p,
                 const double* d_noise_all, const double* h_amp, const double* d_mass, double dt,
                 double half_dt, double half_dt_gamma, int64_t* h_out, int32_t* h_blowup);

/* Replica batch of corrected sweeps (mode 0) or bootstraps (mode 1), one
 * persistent CTA per replica slot, for EAM / elementwise coarse potentials.
 * Arrays carry a leading replica dimension: d_Q and d_P (R, N+1, d), the
 * base and jump arrays (R, N, d), d_noise (R, N, L+1, d), d_hist (R, N).  Slot s works on
 * replica h_ridx[s], windows h_m0[s]..h_m1[s]-1; h_state (2 per slot, {num,
 * den} in/out) and h_out4 (4 per slot: nodes done, failing window, failing
 * substep, kind 1 blow-up / 2 non-finite).  Synchronises. */
int pl_sweep_batch(pl_ctx* ctx, pl_pot* coarse, int64_t d, int L, int64_t N, int R_act,
                   const int32_t* h_ridx, const int64_t* h_m0, const int64_t* h_m1,
                   const int32_t* h_include_m0, int mode, double* d_Q, double* d_P,
                   double* d_baseQ, double* d_baseP, const double* d_jumpQ, const double* d_jumpP,
                   const double* d_noise, const double* h_amp, const double* d_mass, double dt,
                   double half_dt, double half_dt_gamma, double expl, double* h_state,
                   int64_t* h_out4, double* d_hist);

/* d_out[i] = d_a[i] - d_b[i]  (jump = f.q - c.q, parareal.py:280). */
int pl_sub(pl_ctx* ctx, int64_t n, const double* d_a, const double* d_b, double* d_out);

/* ---- SIA hop detection (next row after the hot path) ---- */
/* d_label[b] = smallest doubly occupied BCC site (Wigner-Seitz occupancy) of
 * configuration b (B x 3*n_atoms, unwrapped positions, cubic box n_cells*a). */
int pl_sia_sites(pl_ctx* ctx, int64_t B, int n_atoms, int n_cells, double a, const double* d_q,
                 int32_t* d_label);

/* Stream-ordered: *d_out (device int32) = 1 if any neighbour build of pot
 * exceeded its capacity since the last check, else 0; re-arms the flag. */
int pl_pot_overflow_async(pl_ctx* ctx, pl_pot* pot, int32_t* d_out);

/* ---- measurement --------------------------------------------------------- */
/* Record CUDA events around every kernel stage launched by this host thread
 * until pl_prof_end, which synchronises and returns per-stage summed kernel
 * milliseconds and launch counts (stages: 0 neighbour lists, 1 SNAP U,
 * 2 SNAP Z/Y, 3 SNAP dE/dr, 4 SNAP gather, 5 EAM, 6 integrator). */
int pl_prof_begin(pl_ctx* ctx);
int pl_prof_end(pl_ctx* ctx, int n_stages, double* h_ms, int64_t* h_n);
/* Dense FP64 FMA throughput of the device, measured (TFLOP/s). */
int pl_fp64_peak(pl_ctx* ctx, double* h_tflops);
/* FP64 tensor-core throughput (mma.sync m8n8k4 f64), measured (TFLOP/s): the
 * ceiling of a DMMA formulation of the Z/Y contraction. */
int pl_dmma_peak(pl_ctx* ctx, double* h_tflops);
/* Diagnostic build only (-DPL_YI_TIMING): per (block, phase, warp) cycles of the
 * last Z/Y launch into h_out (4096 x 24 x 24 int64); returns 1 otherwise. */
int pl_yi_timing(int64_t* h_out);

#ifdef __cplusplus
}
#endif

#endif
