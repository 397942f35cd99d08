/*
 * ccf.h — C-ABI of the B200-native CCF spectral Navier–Stokes hot path
 * (arXiv 2206.04827; drop-in for the reference `cylspec` C++ API).
 *
 * Conventions (identical to the reference, proj/include/cylspec/coeffs.hpp:16-45,
 * proj/include/cylspec/grid.hpp:37-50):
 *   - coefficient tensors: complex<double> interleaved (re, im), index (l*n + k)*m + j,
 *     slice l carries wavenumber w = l - p/2 (slice 0 = unpaired Nyquist);
 *   - grid fields: double, same (l, k, j) order, r_j = cos((m-1-j)pi/(m-1)),
 *     z_k likewise, theta_l = (2l - p) pi / p.
 * Every buffer argument may be HOST memory (pageable or pinned) or DEVICE memory of
 * the context's GPU; the library detects which (cudaPointerGetAttributes) and
 * stages host buffers through device memory. Calls are synchronous with respect
 * to the host, like the reference (value semantics), and run on the context's stream.
 *
 * Status codes mirror the reference exception taxonomy one-to-one
 * (proj/include/cylspec/errors.hpp:10-40); the C++ shim (cylspec_b200.hpp)
 * rethrows the same C++ types.
 *
 * Restrictions of the B200 path (documented in DESIGN.md): m and n even
 * (the reference NS pipeline already requires even m, proj/src/ptns.cpp:185),
 * m, n <= 258 for the single-CTA ADI tile.
 */
#ifndef CCF_H_
#define CCF_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ccf_status {
    CCF_OK = 0,
    CCF_DOMAIN_ERROR = 1,          /* cylspec::DomainError */
    CCF_CONFIG_ERROR = 2,          /* cylspec::ConfigError */
    CCF_SINGULAR_OPERATOR = 3,     /* cylspec::SingularOperatorError{shift_index} */
    CCF_NON_CONVERGENCE = 4,       /* cylspec::NonConvergenceError{residual_history} */
    CCF_NOT_INCOMPRESSIBLE = 5,    /* cylspec::NotIncompressibleError{divergence} */
    CCF_NUMERICAL_ERROR = 6,       /* cylspec::NumericalError */
    CCF_CUDA_ERROR = 7,            /* device / driver failure (no reference analogue) */
    CCF_FIELDFILE_ERROR = 8,       /* cylspec::FieldFileError (io.hpp:17-19) */
    CCF_INTERNAL_ERROR = 9
} ccf_status;

typedef struct ccf_ctx ccf_ctx;
typedef struct ccf_ns_state ccf_ns_state;

/* Context: one grid size, one GPU, one stream; caches shift plans and factors
 * (ModalSolverCache, proj/include/cylspec/solvers.hpp:63-76).
 * flags: bit 0 = Q2 endpoint-relative enclosure pad where the reference
 * intervals overlap (off = reference semantics);
 * bit 1 = execute the reference's ADI shift counts. By default the executed Zolotarev
 * plan is the one for adi_tol / 4 (1-2 more shifts per mode) so that slots finishing
 * just above adi_tol do not trigger a serial restart round; the per-round acceptance
 * test (relative residual <= adi_tol) and the restart logic are unchanged;
 * bit 2 = solve the modal Sylvester systems with the ADI kernel (the reference algorithm,
 * adi.cpp:150-202). By default they are solved exactly by fast diagonalization (four batched
 * FP64 tensor-core products per mode, eigenpairs refined in long double at setup): residual
 * ~1e-15 relative, three orders below adi_tol. */
ccf_status ccf_ctx_create(int m, int n, int p, int device, double adi_tol, int flags, ccf_ctx** out);
ccf_status ccf_ctx_destroy(ccf_ctx* ctx);
/* Use an external cudaStream_t (NULL restores the context's own stream). */
ccf_status ccf_ctx_set_stream(ccf_ctx* ctx, void* stream);
ccf_status ccf_ctx_synchronize(ccf_ctx* ctx);

/* transform.hpp:17-22 — analyze / synthesize (synthesize keeps Re only). */
ccf_status ccf_analyze(ccf_ctx* ctx, const double* values, double* coeffs);
ccf_status ccf_synthesize(ccf_ctx* ctx, const double* coeffs, double* values);

/* calculus.hpp:15-29 on Hermitian (real-field) tensors.
 * op: 0 derivative_r, 1 derivative_z, 2 derivative_theta, 4 divide_r,
 *     5 horizontal_laplacian, 6 laplacian. */
ccf_status ccf_calculus(ccf_ctx* ctx, int op, const double* in, double* out);

/* solvers.hpp:86-94 */
ccf_status ccf_poisson3d(ccf_ctx* ctx, const double* f, double* u);
ccf_status ccf_hpoisson(ccf_ctx* ctx, const double* rhs, double* u);

/* timestep.hpp:34-53 HelmholtzTensorStepper::step:
 *   (1 - kappa * diffusivity * lap) X = sum_i bdf_i hist_i + kappa * forcing
 * hist: nhist tensors, newest first (nhist >= order); forcing may be NULL. */
ccf_status ccf_helmholtz_step(ccf_ctx* ctx, const double* const* hist, int nhist, int order, const double* forcing,
                              double diffusivity, double h, double* out);

/* ptns.hpp:47-70 */
ccf_status ccf_pt_synthesize(ccf_ctx* ctx, const double* lam, const double* gam, double* vr, double* vt, double* vz);
ccf_status ccf_pt_decompose(ccf_ctx* ctx, const double* vr, const double* vt, const double* vz, double* lam,
                            double* gam);
ccf_status ccf_curl_vector(ccf_ctx* ctx, const double* vr, const double* vt, const double* vz, double* or_,
                           double* ot, double* oz);
ccf_status ccf_curl_pt(ccf_ctx* ctx, const double* lam, const double* gam, double* lam_out, double* gam_out);
ccf_status ccf_velocity_from_vorticity(ccf_ctx* ctx, const double* lam_w, const double* gam_w, double* lam_v,
                                       double* gam_v);
ccf_status ccf_nonlinear(ccf_ctx* ctx, const double* lam_v, const double* gam_v, const double* lam_w,
                         const double* gam_w, double* lam_out, double* gam_out);
/* nonlinear_term(v, omega, dealias_two_thirds) (ptns.hpp:68-70; rule ptns.cpp:100-110) */
ccf_status ccf_nonlinear_ex(ccf_ctx* ctx, const double* lam_v, const double* gam_v, const double* lam_w,
                            const double* gam_w, int dealias_two_thirds, double* lam_out, double* gam_out);

/* ptns.hpp:84-127 NSStepper (ramp bootstrap). State lives on the device. */
ccf_status ccf_ns_create(ccf_ctx* ctx, double reynolds, double h, int order, int disable_nonlinear,
                         const double* lam0, const double* gam0, ccf_ns_state** out);
/* NSConfig flags (ptns.hpp:84-94): bit 0 disable_nonlinear (Stokes limit), bit 1 dealias_two_thirds,
 * bit 2 compute_gamma_psi (diagnostic Poisson solve, read with ccf_ns_gamma_psi). */
ccf_status ccf_ns_create_ex(ccf_ctx* ctx, double reynolds, double h, int order, int flags, const double* lam0,
                            const double* gam0, ccf_ns_state** out);
ccf_status ccf_ns_step(ccf_ns_state* st, int nsteps);
/* NSStepper::seed (ptns.hpp:110-112, ptns.cpp:195-203): install a prebuilt history. lam_hist / gam_hist: n_omega
 * coefficient tensors (p*n*m complex128 each, host or device), newest first; nl_lam / nl_gam: n_nonlinear
 * nonlinear-term tensors, newest first, entry i belonging to omega entry i + 1 (the next step pushes N of the
 * newest omega in front, ptns.cpp:232). CCF_DOMAIN_ERROR "NSStepper::seed: empty history" for n_omega < 1; a later
 * step with fewer entries than its BDF order fails with "bdf_rhs: insufficient history for the requested order"
 * (timestep.cpp:41-42). The tensors are stored parity-projected (the Helmholtz step projects its right-hand
 * side, timestep.cpp:75). */
ccf_status ccf_ns_seed(ccf_ns_state* st, int n_omega, const double* const* lam_hist, const double* const* gam_hist,
                       int n_nonlinear, const double* const* nl_lam, const double* const* nl_gam, double time,
                       int steps_taken);
/* NSStepper::velocity(): velocity PT scalars of the current state (fresh psi solve, ptns.cpp:205-215). */
ccf_status ccf_ns_velocity(ccf_ns_state* st, double* lam_v, double* gam_v);
/* NSState::gamma_psi = solve_poisson_3d(-gamma_omega) of the omega the last step started from
 * (ptns.cpp:248-253); CCF_CONFIG_ERROR without the flag, CCF_DOMAIN_ERROR before the first step. */
ccf_status ccf_ns_gamma_psi(ccf_ns_state* st, double* gamma_psi);
ccf_status ccf_ns_get_omega(ccf_ns_state* st, double* lam, double* gam, double* time, int* steps_taken);
ccf_status ccf_ns_destroy(ccf_ns_state* st);

/* Per-mode solver API (solvers.hpp:35-82, ultraop.hpp:40-53) for the context's m x n: ModalSolver(m, n, w, scale,
 * poisson, tol) on the device. Matrices are m x n complex128, column-major (Eigen::MatrixXcd / one CoeffTensor
 * slice), in host memory. ccf_modal_solve = ModalSolver::solve(f_full) on the raw C2 x C2 right-hand side
 * (F = A X B + C X D convention, truncated to the top-left (m-2) x (n-2) block; any parity content; scale 0 with
 * poisson 0 is the mass pair, solvers.cpp:57-62): exact fast diagonalization instead of the ADI iteration.
 * ccf_modal_apply = ModalOperator::apply (ultraop.cpp:83-87), the piece of the lifted boundary data
 * (solvers.cpp:125-140, 160-165). ccf_modal_operator: the dense row-major A (0), B (1), C (2), D (3) of raw().
 * Destroying the context first releases the handle's device data; later calls on the handle then report
 * CCF_INTERNAL_ERROR and ccf_modal_destroy only frees it. */
typedef struct ccf_modal ccf_modal;
ccf_status ccf_modal_create(ccf_ctx* ctx, int w, double scale, int poisson, ccf_modal** out);
ccf_status ccf_modal_solve(ccf_modal* h, const double* f_full, double* x);
ccf_status ccf_modal_apply(ccf_modal* h, const double* x, double* y);
ccf_status ccf_modal_operator(ccf_modal* h, int which, double* dense);
ccf_status ccf_modal_destroy(ccf_modal* h);

/* timestep.hpp:60-111 HeatStepper: (d/dt - alpha lap) T = g with the reference's BDF 1 -> order ramp,
 * homogeneous Dirichlet data. initial / forcing: kind 0 = grid values (p*n*m doubles, analyzed on the
 * device: HeatStepper(config, GridField), step_with_callback), kind 1 = coefficients (CoeffTensor).
 * ccf_heat_step adds kappa * forcing to the BDF right-hand side (timestep.cpp:71-73; NULL = none);
 * the caller evaluates the forcing at t + h (ForcingMode::exact) or t. heat_run (timestep.cpp:146-170)
 * is this loop plus synthesize() of the snapshots (C++ shim, Python mirror). Destroy with ccf_ns_destroy. */
ccf_status ccf_heat_create(ccf_ctx* ctx, double alpha, double h, int order, const double* initial, int initial_kind,
                           ccf_ns_state** out);
ccf_status ccf_heat_step(ccf_ns_state* st, const double* forcing, int forcing_kind);
ccf_status ccf_heat_get(ccf_ns_state* st, double* coeffs, double* time, int* steps_taken);

/* Mode sharding of the NS / heat stepper over the GPUs of one node (the reference is
 * single-process, ptns.cpp:217-267 — this replaces nothing, it partitions NSStepper::step).
 * Rank r of world computes the half-spectrum Fourier slots [slot_lo, slot_hi) (w = slot, slot p/2 =
 * Nyquist) in every per-mode stage and the radial value rows [row_lo, row_hi) of all slots in the
 * theta stage, reading / writing each slot's values in the owning rank's exchange buffer through
 * peer memory (NVLink), ordered by two rank barriers per step. Every rank passes the full initial
 * field to ccf_ns_create; ccf_ns_get_omega fills the rank's own slots (w = +-slot) correctly and
 * leaves the others meaningless: gather by slot ownership. Call order: ccf_ctx_create ->
 * ccf_shard_init -> (ccf_shard_ipc_handle, exchange the handles, ccf_shard_open_ipc)
 * | ccf_shard_link_local -> ccf_ns_create. Other compute entry points on a sharded context return
 * CCF_CONFIG_ERROR. world == 1 leaves the context unsharded. */
ccf_status ccf_shard_init(ccf_ctx* ctx, int rank, int world);
/* Host-only (no GPU): the partition ccf_shard_init uses, world + 1 bounds each
 * (rank r: slots [slot_bounds[r], slot_bounds[r+1]), rows [row_bounds[r], row_bounds[r+1])). */
ccf_status ccf_shard_partition(int m, int p, int world, int* slot_bounds, int* row_bounds);
ccf_status ccf_shard_info(ccf_ctx* ctx, int* rank, int* world, int* slot_lo, int* slot_hi, int* row_lo, int* row_hi);
/* CCF_SHARD_HANDLE_BYTES-byte handle of this rank's exchange buffer (CUDA IPC handle + offset). */
#define CCF_SHARD_HANDLE_BYTES 128
ccf_status ccf_shard_ipc_handle(ccf_ctx* ctx, void* handle);
/* world x CCF_SHARD_HANDLE_BYTES bytes of handles in rank order (own entry ignored): maps the peers' exchange buffers;
 * rank barriers then run on the device (graph-capturable). */
ccf_status ccf_shard_open_ipc(ccf_ctx* ctx, const void* handles);
/* Ranks emulated in one process on one device (contexts ctxs[r] sharded as rank r of world): peer
 * buffers are plain device pointers and the barriers are host barriers between the threads that
 * step the ranks concurrently (no device-side waiting between ranks). */
ccf_status ccf_shard_link_local(ccf_ctx* const* ctxs, int world);
/* Replace the device barrier by stream synchronisation + fn(user) (a host barrier across ranks);
 * fn == NULL restores the device barrier. */
ccf_status ccf_shard_set_host_barrier(ccf_ctx* ctx, void (*fn)(void*), void* user);

/* CCF1 FieldFile I/O (io.hpp:11-28, io.cpp:12-109): "CCF1" | version u32 = 1 | kind u8 (0 real grid
 * values, m*n*p doubles; 1 complex coefficients, 2*m*n*p doubles interleaved) | m, n, p u32 |
 * payload f64 LE in (l, k, j) order | CRC-32/IEEE of the payload bytes. Payloads may be host or
 * device memory; device payloads are checksummed on the GPU (only the file bytes cross PCIe).
 * Errors (FieldFileError: bad magic, unsupported version, unknown kind, truncation, CRC mismatch,
 * open/write failures) return CCF_FIELDFILE_ERROR with the reference's message in ccf_create_error. */
ccf_status ccf_write_field(const char* path, int kind, int m, int n, int p, const double* payload);
ccf_status ccf_read_field_header(const char* path, int* kind, int* m, int* n, int* p);
/* payload: cap doubles of host or device memory (>= the file's count) */
ccf_status ccf_read_field(const char* path, int* kind, int* m, int* n, int* p, double* payload, size_t cap);
/* crc32_ieee (io.cpp:12-25) of host or device bytes (device: on the GPU) */
ccf_status ccf_crc32(const void* data, size_t len, unsigned* crc);
/* Snapshot of the stepper's omega (lambda, gamma) as kind-1 FieldFiles, written from the device
 * state (cylspec_main.cpp:111-113 writes snapshots with write_field); NULL path skips one. */
ccf_status ccf_ns_write_omega(ccf_ns_state* st, const char* lam_path, const char* gam_path);

/* Details of the last error on this context (thread-compatible, not thread-safe).
 * kind = ccf_status; slice = Fourier slice of a failed modal solve or -1;
 * shift_index = ADI shift of a singular operator or -1; residual history of a
 * NonConvergenceError (up to *n_hist entries on input). */
ccf_status ccf_get_last_error(ccf_ctx* ctx, int* kind, int* slice, int* shift_index, double* residual_hist,
                              int* n_hist, char* msg, int cap);

/* Statistics since the last reset: ADI solves, iterations executed (J x rounds),
 * max rounds, worst final residual; kernel launches issued. */
ccf_status ccf_get_stats(ccf_ctx* ctx, long* adi_subproblems, long* adi_iterations, int* max_rounds,
                         double* worst_residual, long* kernel_launches);
ccf_status ccf_reset_stats(ccf_ctx* ctx);
/* FP64 tensor-core flops (2 M N K per product term) of the batched GEMMs enqueued since the last
 * ccf_reset_stats (host-side count: steps replayed from a CUDA graph are not counted). */
ccf_status ccf_get_gemm_flops(ccf_ctx* ctx, double* flops);
/* Per (tensor, slot) ADI rounds used (1..4) and relative residual after each round
 * (history[4 * i + r]) of the most recent ADI solve on this context (adi.cpp:163-200):
 * which = 0 most recent solve, 1 / 2 most recent Poisson / Helmholtz solve (needs
 * ccf_adi_keep_history(ctx, 1) beforehand; adds two device copies per solve). */
ccf_status ccf_adi_keep_history(ccf_ctx* ctx, int enable);
ccf_status ccf_adi_last_rounds(ccf_ctx* ctx, int which, int* ntensor, int* nslots, int* rounds, double* history,
                               int cap);

/* Shift plan of the (|w|, poisson|scale) modal solver of this context (for parity
 * tests against the reference plan): info = {a, b, c, d, gamma, alpha, modulus, J}. */
ccf_status ccf_modal_plan(ccf_ctx* ctx, int w, double scale, int poisson, double* info, double* u, double* v,
                          int cap);

/* Benchmark / profiling helpers: enable CUDA-graph replay of steady-state steps (default on),
 * report kernel launches per steady-state step, and run the next step eagerly with CUDA events
 * at the stage boundaries (P Poisson ADI, V pt_synthesize, X1 r,z synthesis, X2 theta x cross,
 * X3 r,z analysis, C curl + decompose, H Helmholtz ADI). */
ccf_status ccf_ns_set_graphs(ccf_ns_state* st, int enable);
ccf_status ccf_ns_launches_per_step(ccf_ns_state* st, long* n);
ccf_status ccf_ns_profile_step(ccf_ns_state* st, double* ms, int* nstages, char* names, int cap);

/* Host-only (no GPU) modal shift plan with the context's setup numerics; error text via ccf_create_error.
 * info[0..7] = (a, b, c, d, gamma, alpha, modulus, J); flags bit0 = Q2 endpoint pad, bit1 = also
 * report info[8] = 1 if a banded LU of this slot pivots (caller then provides info[9]). */
ccf_status ccf_plan_host(int m, int n, int w, double scale, int poisson, double tol, int flags, double* info, double* u,
                         double* v, int cap);

/* Host-only (no GPU) check of the fast-diagonalization solver data of one mode: relative residual
 * ||A X B + C X D - E|| / ||E|| (long double) of the device arithmetic (four double products) on a
 * seeded random RHS, for wavenumber w, k-parity k0, Poisson or Helmholtz(scale). */
ccf_status ccf_diag_host_check(int m, int n, int w, double scale, int poisson, int k0, unsigned long long seed,
                               double* residual);

/* Message of the last failed ccf_ctx_create / ccf_plan_host on this thread. */
const char* ccf_create_error(void);
const char* ccf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CCF_H_ */
