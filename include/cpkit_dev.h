/*
 * cpkit_dev.h - device-level C ABI of the B200 build.
 *
 * The reference has no device layer; these entry points expose the
 * internal C++ seams of its solver path one by one so each
 * can be checked against the CPU oracle and timed with device-resident
 * inputs. Each entry cites the reference function whose semantics it keeps.
 * Error convention and status codes are those of cpkit.h.
 *
 * A cpkit_dev_problem owns, on one GPU: the (slab of the) tensor, the
 * replicated factors, the dimension-tree cache and every GN/ALS buffer.
 * Factor blocks cross the boundary as ONE stacked row-major buffer:
 * mode 0 (s_0 x R), then mode 1, ... (sum_n s_n * R doubles).
 */
#ifndef CPKIT_DEV_H
#define CPKIT_DEV_H

#include "cpkit.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cpkit_dev_problem cpkit_dev_problem;

/* Problem of global extents dims[order] at rank R on CUDA device `device`. */
CPKIT_API cpkit_status cpkit_dev_problem_create(int device, const uint64_t* dims, uint64_t order,
                                                uint64_t rank, cpkit_dev_problem** out);
/* Last-mode sharded problem: this process owns slab `shard` of `world`
 * (NCCL communicator from a 128-byte unique id made by
 * cpkit_dev_nccl_unique_id on shard 0 and broadcast by the caller). */
CPKIT_API cpkit_status cpkit_dev_nccl_unique_id(void* out128);
CPKIT_API cpkit_status cpkit_dev_problem_create_sharded(int device, const uint64_t* dims, uint64_t order,
                                                        uint64_t rank, int shard, int world,
                                                        const void* nccl_id128,
                                                        cpkit_dev_problem** out);
/* TEST ONLY: `world` last-mode shards of one problem on ONE device, joined by
 * an in-process loopback group instead of NCCL (collectives become device
 * copies and a fixed rank-order sum; ranks meet on the host). Fills out[0..world).
 * Each shard must be driven by its own host thread, issuing the same call
 * sequence on every shard, exactly as NCCL ranks would. Lets one GPU run the
 * sharded code path of a multi-GPU job. */
CPKIT_API cpkit_status cpkit_dev_problem_create_loopback(int device, const uint64_t* dims, uint64_t order,
                                                         uint64_t rank, int world, cpkit_dev_problem** out);
CPKIT_API void cpkit_dev_problem_destroy(cpkit_dev_problem* p);
/* [lo, hi) rows of the last mode owned by this problem, and its element count. */
CPKIT_API cpkit_status cpkit_dev_slab(const cpkit_dev_problem* p, uint64_t* lo, uint64_t* hi,
                                      uint64_t* local_elems);

/* Tensor in: host copy of the local slab (tensor.hpp:16-48 layout). */
CPKIT_API cpkit_status cpkit_dev_upload_tensor(cpkit_dev_problem* p, const double* host_local);
/* Tensor in from a CPKT1 file (tensor.cpp:197-239), streamed: chunks of whole
 * last-mode rows are read into two pinned staging buffers while the previous
 * chunk is copied to HBM (only this shard's slab columns); the finiteness
 * check of the reference's read_tensor runs on the device. No host copy of
 * the tensor is made. */
CPKIT_API cpkit_status cpkit_dev_load_tensor(cpkit_dev_problem* p, const char* path);
/* Tensor generated on device: reconstruct(truth) (kruskal.cpp:67-92, bitwise)
 * plus keyed-RNG Gaussian noise scaled to noise_rel * ||X||_F. */
CPKIT_API cpkit_status cpkit_dev_generate_tensor(cpkit_dev_problem* p, const double* truth_factors,
                                                 uint64_t noise_seed, double noise_rel);
CPKIT_API cpkit_status cpkit_dev_set_factors(cpkit_dev_problem* p, const double* factors);
CPKIT_API cpkit_status cpkit_dev_get_factors(cpkit_dev_problem* p, double* factors);

/* ||X||^2 (tensor.cpp:61-67). */
CPKIT_API cpkit_status cpkit_dev_norm2(cpkit_dev_problem* p, double* out);
/* Dimension-tree MTTKRP with workspace reuse (mttkrp.cpp:160-189); out may
 * be NULL (result stays on device for cpkit_dev_residual). */
CPKIT_API cpkit_status cpkit_dev_mttkrp(cpkit_dev_problem* p, uint64_t mode, double* out);
/* Uncached MTTKRP (mttkrp.cpp:149-158). */
CPKIT_API cpkit_status cpkit_dev_mttkrp_naive(cpkit_dev_problem* p, uint64_t mode, double* out);
/* MttkrpWorkspace::note_factor_update / full_contractions (mttkrp.hpp:40-45). */
CPKIT_API cpkit_status cpkit_dev_note_factor_update(cpkit_dev_problem* p, uint64_t mode);
CPKIT_API int cpkit_dev_full_contractions(const cpkit_dev_problem* p);
CPKIT_API void cpkit_dev_reset_contraction_counter(cpkit_dev_problem* p);

/* GammaSet from the current factors (kruskal.cpp:42-65); grams N*R*R,
 * pairwise N*N*R*R ([n][p] blocks). Either output may be NULL. */
CPKIT_API cpkit_status cpkit_dev_gamma_set(cpkit_dev_problem* p, double* grams, double* pairwise);
/* Replace the device GammaSet (reference tests use hand-built sets). */
CPKIT_API cpkit_status cpkit_dev_set_gamma_set(cpkit_dev_problem* p, const double* grams,
                                               const double* pairwise);
/* residual_fitness (kruskal.cpp:94-118) from the device M^(N-1) and the
 * device grams of the current factors. */
CPKIT_API cpkit_status cpkit_dev_residual(cpkit_dev_problem* p, double xnorm2, double* r, double* f);
/* gradient (gauss_newton.cpp:81-94): mttkrps stacked (NULL = device M). */
CPKIT_API cpkit_status cpkit_dev_gradient(cpkit_dev_problem* p, const double* mttkrps, double* g_out);
/* hessian_matvec (gauss_newton.cpp:96-136); shape 0 identity, 1 diagonal. */
CPKIT_API cpkit_status cpkit_dev_jtj_matvec(cpkit_dev_problem* p, const double* w, double lambda,
                                            int shape, double* u_out);
/* build_preconditioner (gauss_newton.cpp:190-207): N*R*R inverses. */
CPKIT_API cpkit_status cpkit_dev_preconditioner(cpkit_dev_problem* p, double lambda, int shape,
                                                double* out);
/* cp_cg (gauss_newton.cpp:279-349); gn_config_json as the "gn" block of
 * cpkit_decompose (NULL = defaults). */
CPKIT_API cpkit_status cpkit_dev_cp_cg(cpkit_dev_problem* p, const double* g, double lambda,
                                       const char* gn_config_json, double* v_out, int* iterations,
                                       int* hit_cap, int* breakdown);
/* spd_solve / spd_inverse (matrix_ops.cpp:60-81) on an R x R system. */
CPKIT_API cpkit_status cpkit_dev_spd_solve(cpkit_dev_problem* p, const double* s, const double* b,
                                           uint64_t rows, double lambda, double* y_out);
CPKIT_API cpkit_status cpkit_dev_spd_inverse(cpkit_dev_problem* p, const double* s, double lambda,
                                             double* inv_out);
/* als_sweep (als.cpp:22-52): factors updated on device. */
CPKIT_API cpkit_status cpkit_dev_als_sweep(cpkit_dev_problem* p, double lambda, double* step_norm,
                                           int* full_contractions);
/* gn_step (gauss_newton.cpp:360-449) with a fresh schedule from the config;
 * diag12 = [halt, stepped, residual_before, residual_after, grad_norm,
 * lambda, cg_iters, step_norm, alpha, armijo_exhausted, cg_hit_cap,
 * cg_breakdown]. */
CPKIT_API cpkit_status cpkit_dev_gn_step(cpkit_dev_problem* p, const char* gn_config_json,
                                         double xnorm2, double* diag12);
/* als_optimize / gn_optimize on the resident tensor (config as
 * cpkit_decompose's, "optimizer" selects); init/out factors stacked. */
CPKIT_API cpkit_status cpkit_dev_optimize(cpkit_dev_problem* p, const char* config_json,
                                          const double* init_factors, double* out_factors,
                                          cpkit_report** out_report);

/* ---- timing (CUDA events on the problem's stream; milliseconds) ---- */
/* `sweeps` back-to-back ALS sweeps at lambda (factors evolve). */
CPKIT_API cpkit_status cpkit_dev_time_als_sweeps(cpkit_dev_problem* p, double lambda, int sweeps,
                                                 double* ms_total);
/* reps x (back root, front root) root-GEMM launches; average ms per launch each. */
CPKIT_API cpkit_status cpkit_dev_time_roots(cpkit_dev_problem* p, int reps, double* ms_back,
                                            double* ms_front);
/* Per-launch event timing of the dominant kernels inside a caller's timed
 * region: kinds [0] back-root GEMM, [1] front-root GEMM (+ split-K reduce),
 * [2] persistent CG solve. enable(1) clears the record. */
CPKIT_API cpkit_status cpkit_dev_profile(cpkit_dev_problem* p, int enable);
CPKIT_API cpkit_status cpkit_dev_profile_read(cpkit_dev_problem* p, double* ms3, int* count3);
/* reps x J^T J v on the current factors; average ms per matvec. */
CPKIT_API cpkit_status cpkit_dev_time_jtj(cpkit_dev_problem* p, int reps, double* ms);
/* reps x ||X||^2 streaming pass; average ms. */
CPKIT_API cpkit_status cpkit_dev_time_norm2(cpkit_dev_problem* p, int reps, double* ms);
/* reps x the second dimension-tree level (mttkrp.cpp:63-75: M^(0) from the cached
 * back-root partial, an HBM-bound pass); average ms and the partial's bytes. */
CPKIT_API cpkit_status cpkit_dev_time_second_level(cpkit_dev_problem* p, int reps, double* ms, double* bytes);
/* FP64 DMMA issue-rate probe on `device`, TFLOP/s (roofline denominator). */
CPKIT_API cpkit_status cpkit_dev_probe_dmma_peak(int device, double* tflops);
/* `steps` gn_step calls (one schedule from the config); total ms and the
 * inner CG iterations they ran. */
CPKIT_API cpkit_status cpkit_dev_time_gn_steps(cpkit_dev_problem* p, const char* gn_json, int steps,
                                               double* ms, int* cg_iters_total);
/* Seeded inputs: generators.cpp:59-76 factor draws (kind 0 uniform(a,b),
 * 1 gaussian) and harness.cpp:378-391 seed derivations. */
CPKIT_API cpkit_status cpkit_dev_random_factors(const uint64_t* dims, uint64_t order, uint64_t rank,
                                                uint64_t seed, int kind, double a, double b,
                                                double* out);
CPKIT_API uint64_t cpkit_dev_problem_seed(uint64_t master, int rank, int problem);
CPKIT_API uint64_t cpkit_dev_init_seed(uint64_t master, int rank, int problem, int init);
/* Rows [lo, hi) of a last-mode extent owned by `shard` of `world` (the
 * balanced contiguous split used by cpkit_dev_problem_create_sharded). */
CPKIT_API cpkit_status cpkit_dev_shard_range(uint64_t extent, int shard, int world, uint64_t* lo,
                                             uint64_t* hi);
/* Device tensor slab back to host. */
CPKIT_API cpkit_status cpkit_dev_download_tensor(cpkit_dev_problem* p, double* host_local);
/* Number of kernels this library launched since load (for the bench). */
CPKIT_API uint64_t cpkit_dev_kernel_launches(void);
/* Guarded allocation mode (env CPKIT_GUARD=1, the pool has no compute-sanitizer):
 * device buffers released so far whose 64 KB red zones were overwritten. */
CPKIT_API uint64_t cpkit_dev_guard_violations(void);
/* Positive control of the guard mode: out-of-bounds writes past both ends of
 * fresh buffers are detected (*detected = 1). INVALID_ARGUMENT without CPKIT_GUARD. */
CPKIT_API cpkit_status cpkit_dev_guard_selftest(int* detected);

#ifdef __cplusplus
}
#endif

#endif /* CPKIT_DEV_H */
