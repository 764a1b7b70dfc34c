/*
 * yasps_b200.h — C-ABI of the B200-native YASPS Newton-step hot path.
 *
 * This is the drop-in boundary under the reference's C++ `relsim::Engine`
 * (/root/reference/proj/include/relsim/engine.hpp:27-80).  Every entry point
 * takes plain pointers and sizes; host pointers are only borrowed for the
 * duration of a call.  Device state lives in an opaque context.
 *
 * The reference has no FFI: its seam is the C++ class `Engine` plus the
 * scene/energy builders that record what each energy term is.  The mapping
 * of each entry point to the reference interface it replaces is given in the
 * comment above it.  INTEGRATION.md shows the C++ shim a maintainer adds on
 * the reference side.
 *
 * Error model (reference: core.hpp:33-71, README.md:38-39): every function
 * returns YS_OK (0) or a non-zero status whose class mirrors the reference's
 * exception hierarchy; ys_last_error() returns the message text, worded like
 * the reference's (tests match on "stale", "iteration", "[3, 6)", ...).
 *
 * The oracle under oracle/ exports the same functions with the prefix `yo_`
 * (CPU restatement, test infrastructure only).
 */
#ifndef YASPS_B200_H
#define YASPS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes / error classes (core.hpp:33-71) ---------------------- */
#define YS_OK 0
#define YS_ERR_VALIDATION 1 /* relsim::ValidationError (UserError, exit 2) */
#define YS_ERR_DECL 2       /* relsim::DeclError       (UserError, exit 2) */
#define YS_ERR_NUMERICAL 3  /* relsim::NumericalError  (exit 3)            */
#define YS_ERR_INTERNAL 4   /* relsim::InternalError                       */
#define YS_ERR_CUDA 5       /* device / driver failure (no reference twin) */

/* ---- projection modes (scene.hpp:153) ----------------------------------- */
#define YS_PROJECT_FULL 0    /* ProjectionMode::FullProject    */
#define YS_PROJECT_REDUCED 1 /* ProjectionMode::ReducedProject */

/* ---- point-domain kinds: how a 3-D point maps to target DoFs ------------
 * sim.cpp:231-235 (free), 236-252 (affine body), 288-294 (fixed).          */
#define YS_POINTS_FREE 0
#define YS_POINTS_AFFINE 1
#define YS_POINTS_FIXED 2

typedef struct ys_context ys_context;

/* StepStats (engine.hpp:15-21) + PcgResult (solver.hpp:33-40). */
typedef struct ys_step_stats {
  int64_t pcg_iterations;
  double pcg_residual;  /* ||r|| / ||g|| at exit                          */
  int32_t pcg_converged;
  int32_t regularized_blocks; /* BlockJacobiPreconditioner::regularized_ */
  double assemble_seconds;    /* refresh_dynamic + assemble (engine.cpp:76-81) */
  double solve_seconds;       /* preconditioner build + PCG                */
} ys_step_stats;

/* ------------------------------------------------------------------------
 * Context lifecycle
 * ------------------------------------------------------------------------ */
int ys_create(ys_context** out, int32_t device);
void ys_destroy(ys_context* ctx);
const char* ys_last_error(const ys_context* ctx);
int ys_last_error_class(const ys_context* ctx);
/* Library build string (arch, version) — lets a caller prove which .so ran. */
const char* ys_version(void);

/* ------------------------------------------------------------------------
 * Minimize targets -> GradientLayout (index_gen.hpp:14-30, index_gen.cpp:22-38)
 * Targets are registered in Scene::add_minimize_target order (scene.cpp:326-334);
 * each owns instances*rc contiguous DoFs.
 * ------------------------------------------------------------------------ */
int ys_add_target(ys_context* ctx, int64_t instances, int32_t rc, int32_t* target_id);
/* Attribute::update_value on a target (values: instances*rc, row-major). */
int ys_set_target_values(ys_context* ctx, int32_t target, const double* values);
int ys_get_target_values(ys_context* ctx, int32_t target, double* values);
int ys_total_dofs(ys_context* ctx, int64_t* s);

/* ------------------------------------------------------------------------
 * Point domains: the parameterisations a UNION joins (sim.cpp:223-294).
 *   FREE   : position is target `target_a` itself (rc 3), n = its instances.
 *   AFFINE : p_i = A[v2b[i]] * rest_i + t[v2b[i]], A = target_a (rc 9,
 *            row-major), t = target_b (rc 3); rest: n x 3.
 *   FIXED  : constant positions (n x 3); contributes no DoFs.
 * ------------------------------------------------------------------------ */
int ys_add_points(ys_context* ctx, int32_t kind, int64_t n, int32_t target_a, int32_t target_b,
                  const int64_t* v2b, const double* rest_or_positions, int32_t* domain_id);
/* Current point positions of a domain (evaluates A r + t for affine). */
int ys_get_points(ys_context* ctx, int32_t domain, double* positions);

/* PrimitiveUnion over point domains (scene.hpp:121-139, scene.cpp:205-237). */
int ys_add_point_union(ys_context* ctx, int32_t n_children, const int32_t* domains,
                       int32_t* union_id);

/* Pair primitive with an arity-2 connectivity into a union (sim.cpp:445-447).
 * dynamic=1 marks a dynamic primitive (PrimitiveType(..., is_dynamic)). */
int ys_add_pair_set(ys_context* ctx, int32_t union_id, int32_t dynamic, int32_t* pairset_id);
/* A stencil primitive of arity 2, 3 or 4 into a union (a pair set is arity 2):
 * the point-edge (3) and point-triangle / edge-edge (4) barriers below.  Not in
 * the reference (its contact is point-point only, proj/README.md:110-111). */
int ys_add_stencil_set(ys_context* ctx, int32_t union_id, int32_t arity, int32_t dynamic, int32_t* set_id);
/* Candidate primitives of a contact stencil set (not in the reference):
 * kind 1 PT (prims_a: n_a points, prims_b: n_b triangles of 3 points),
 * kind 2 EE (prims_a: n_a edges of 2 points; self-contact, prims_b ignored),
 * kind 3 PE (prims_a: n_a points, prims_b: n_b edges); union indices. */
int ys_set_stencil_primitives(ys_context* ctx, int32_t set, int32_t kind, int64_t n_a, const int64_t* prims_a,
                              int64_t n_b, const int64_t* prims_b);
/* The contact candidates on the device: every (a, b) (EE: b > a) sharing no
 * point, not all points fixed, with the squared distance of its IPC distance
 * type strictly below dhat, in (a, b) order; then resize_dynamic. */
int ys_refresh_stencils(ys_context* ctx, int32_t set, double dhat, int64_t* n_stencils);
/* PrimitiveType::resize_dynamic (scene.cpp:171-199): replaces the pair table
 * (arity*n union-global indices; 2*n for pair sets) and bumps the dynamic epoch. Static pair sets
 * may only be set before ys_finalize. */
int ys_set_pairs(ys_context* ctx, int32_t pairset, int64_t n, const int64_t* pairs);
int ys_pair_count(ys_context* ctx, int32_t pairset, int64_t* n);
/* The current pair table (2*n union-global indices). */
int ys_get_pairs(ys_context* ctx, int32_t pairset, int64_t* pairs);
/* Simulation::refresh_dynamic_pairs (sim.cpp:456-484) on the device: every
 * pair (i in child ca, j in child cb), ca < cb, not both fixed, with squared
 * distance < dhat, in the reference's loop order; then resize_dynamic. */
int ys_refresh_pairs(ys_context* ctx, int32_t pairset, double dhat,
                     const int32_t* child_is_fixed, int64_t* n_pairs);

/* ------------------------------------------------------------------------
 * Energies (energies.hpp:20-54).  Each call records one term group with a
 * kind tag; the symbolic JOIN/UNION layout it implies is fixed by the kind.
 * `weight` is the per-instance scale (dt^2 in the driver, sim.cpp:193-194).
 * ------------------------------------------------------------------------ */
/* add_stable_neo_hookean (energies.cpp:49-118). rest: the target's rest
 * positions (instances x 3). via_deformation_gradient=1 -> ReducedProject. */
int ys_add_stable_neo_hookean(ys_context* ctx, int32_t pos_target, int64_t n_tets,
                              const int64_t* t2v, const double* rest_positions,
                              double youngs_modulus, double poisson_ratio, double weight,
                              int32_t via_deformation_gradient, int32_t* energy_id);
/* add_point_point_barrier (energies.cpp:30-47): kappa (d-dhat)^2 log(d/dhat)^2,
 * d squared distance, over a pair set. */
int ys_add_point_point_barrier(ys_context* ctx, int32_t pairset, double dhat, double kappa,
                               double weight, int32_t mode, int32_t* energy_id);
/* Point-triangle (stencil p, t0, t1, t2), edge-edge (a0, a1, b0, b1) and
 * point-edge (p, e0, e1) barriers — NOT IN THE REFERENCE: weight kappa
 * (d - dhat)^2 log(d / dhat)^2 (the point-point barrier of energies.cpp:30-47)
 * on the squared distance d between the primitives, with IPC's distance types
 * (point-plane / line-line / point-line / point-point by the closest-point
 * region), FullProject.  Stencil sets of arity 4 / 4 / 3 over unions of free
 * and fixed points. */
int ys_add_point_triangle_barrier(ys_context* ctx, int32_t set, double dhat, double kappa, double weight,
                                  int32_t* energy_id);
int ys_add_edge_edge_barrier(ys_context* ctx, int32_t set, double dhat, double kappa, double weight,
                             int32_t* energy_id);
int ys_add_point_edge_barrier(ys_context* ctx, int32_t set, double dhat, double kappa, double weight,
                              int32_t* energy_id);
/* add_repulsive_energy (energies.cpp:20-28): weight / ||p0 - p1||. */
int ys_add_repulsive(ys_context* ctx, int32_t pairset, double weight, int32_t mode,
                     int32_t* energy_id);
/* add_inertia (energies.cpp:168-174) over a point domain: 0.5 m |x - x~|^2. */
int ys_add_inertia(ys_context* ctx, int32_t domain, const double* mass, const double* x_tilde,
                   int32_t* energy_id);
/* x_tilde update (Simulation::begin_frame, sim.cpp:488-500). */
int ys_set_inertia_anchor(ys_context* ctx, int32_t energy, const double* x_tilde);
/* add_affine_orthogonality (energies.cpp:120-127): 0.5 k w ||A^T A - I||_F^2. */
int ys_add_affine_orthogonality(ys_context* ctx, int32_t amat_target, double stiffness,
                                double weight, int32_t* energy_id);
/* add_bending (energies.cpp:129-155): k w l0 ||n1^ - n2^|| over hinges. */
int ys_add_bending(ys_context* ctx, int32_t pos_target, int64_t n_hinges, const int64_t* h2v,
                   const double* rest_positions, double stiffness, double weight,
                   int32_t* energy_id);

/* ------------------------------------------------------------------------
 * Engine (engine.hpp:27-80)
 * ------------------------------------------------------------------------ */
/* Engine::Engine (engine.cpp:7-20): builds the static structures and the
 * dynamic ones for the current pair tables. */
int ys_finalize(ys_context* ctx);
/* Engine::refresh_dynamic / dynamic_stale (engine.cpp:41-45). */
int ys_refresh_dynamic(ys_context* ctx);
int ys_dynamic_stale(ys_context* ctx, int32_t* stale);
/* Engine::assemble(project, with_hessian) (engine.cpp:47-60). */
int ys_assemble(ys_context* ctx, int32_t project, int32_t with_hessian);
/* Engine::gradient(). */
int ys_get_gradient(ys_context* ctx, double* g);
/* Engine::total_energy (engine.cpp:64-68); sum over energies in declaration
 * order. A log of a non-positive value raises YS_ERR_NUMERICAL. */
int ys_total_energy(ys_context* ctx, double* energy);
/* Per-energy totals, in declaration order (Evaluator::total, eval.cpp:394-401). */
int ys_energy_totals(ys_context* ctx, double* totals);
/* Engine::apply_hessian (engine.cpp:70-73): y += (H_static + H_dynamic) x. */
int ys_apply_hessian(ys_context* ctx, const double* x, double* y);
/* Engine::minimize_step (engine.cpp:75-101): refresh_dynamic, assemble, block
 * Jacobi, PCG(tol, max_iter<0 -> max(2s, 64)). dx (may be NULL: result stays
 * on the device) receives the unnegated solution, targets in registration
 * order. */
int ys_minimize_step(ys_context* ctx, double tol, int64_t max_iter, double* dx,
                     ys_step_stats* stats);
/* PCG residual history of the last solve (||r||/||g|| per iteration, 1.0 first). */
int ys_pcg_history(ys_context* ctx, int64_t capacity, double* history, int64_t* count);
/* Engine::gather_targets / scatter_targets (engine.cpp:103-120). */
int ys_gather_targets(ys_context* ctx, double* x);
int ys_scatter_targets(ys_context* ctx, const double* x);
/* Device-resident line-search update: X = X0 - alpha * dx_last, X0 being the
 * state at the last minimize_step (sim.cpp:546).  alpha == 0 restores X0. */
int ys_step_targets(ys_context* ctx, double alpha, double* max_abs_step);

/* ------------------------------------------------------------------------
 * Introspection used by the parity tests and tooling
 * ------------------------------------------------------------------------ */
/* which: 0 = static_hessian(), 1 = dynamic_hessian() (BlockSparseHessian,
 * assembly.hpp:19-60). checksum = structure_checksum (assembly.cpp:136-153). */
int ys_hessian_info(ys_context* ctx, int32_t which, int64_t* n_groups, int64_t* n_blocks,
                    int64_t* n_values, uint64_t* checksum);
/* groups: n_groups x 5 int64 {rows, cols, coord_start, count, value_start}. */
int ys_hessian_groups(ys_context* ctx, int32_t which, int64_t* groups);
int ys_hessian_coords(ys_context* ctx, int32_t which, int64_t* row, int64_t* col);
int ys_hessian_values(ys_context* ctx, int32_t which, double* values);
/* CompiledEnergy tables (assembly.hpp:75-103). */
int ys_energy_info(ys_context* ctx, int32_t energy, int64_t* instances, int32_t* kappa,
                   int32_t* width, int32_t* dynamic);
/* instances x kappa SlotEntry {index (1-based, 0 pad), len, col} (index_gen.hpp:61-65). */
int ys_energy_slots(ys_context* ctx, int32_t energy, int64_t* index, int32_t* len, int32_t* col);
/* Compressed dimension m per instance (InstancePlan::m). */
int ys_energy_compressed_sizes(ys_context* ctx, int32_t energy, int32_t* m);
/* DiagAccumulator blocks (assembly.hpp:63-71), concatenated in target-instance
 * order, each rc x rc row-major. */
int ys_diag_blocks(ys_context* ctx, double* blocks);
/* Device memory in use by the context, bytes. */
int ys_device_bytes(ys_context* ctx, int64_t* bytes);

/* ------------------------------------------------------------------------
 * Free-standing solver entry points over a caller-built BSR, mirroring
 * BlockSparseHessian::build + spmv_add + BlockJacobi + pcg (solver.hpp:13-48).
 * coords: n x 4 int64 {rows, cols, row, col}; duplicate coordinates merge.
 * ------------------------------------------------------------------------ */
int ys_bsr_build(ys_context* ctx, int64_t total_dofs, int64_t n_coords, const int64_t* coords,
                 int32_t* bsr_id);
int ys_bsr_info(ys_context* ctx, int32_t bsr, int64_t* n_groups, int64_t* n_blocks,
                int64_t* n_values, uint64_t* checksum);
int ys_bsr_groups(ys_context* ctx, int32_t bsr, int64_t* groups);
int ys_bsr_coords(ys_context* ctx, int32_t bsr, int64_t* row, int64_t* col);
int ys_bsr_set_values(ys_context* ctx, int32_t bsr, const double* values);
/* y += H x (spmv_add, solver.cpp:59-82). */
int ys_bsr_spmv(ys_context* ctx, int32_t bsr, const double* x, double* y);
/* pcg(h, g, BlockJacobi(diag blocks of width bs), tol, max_iter) (solver.cpp:151-205);
 * bs = 0 selects the identity preconditioner. */
int ys_bsr_pcg(ys_context* ctx, int32_t bsr, int32_t bs, const double* g, double tol,
               int64_t max_iter, double* x, int64_t* iterations, double* rel_residual,
               int32_t* converged);

/* ------------------------------------------------------------------------
 * Multi-GPU: row-partitioned PCG, one process per GPU.
 * Every rank registers the same scene, so structures, evaluation and assembly
 * are replicated; minimize_step then solves with each rank owning a
 * contiguous range of block rows (balanced by stored entries), exchanging the
 * halo of p once per iteration and the dot-product partials of every rank
 * twice per iteration.  Partials are summed in rank order on every rank, so
 * all ranks hold bit-identical alpha / beta / status and stop together; the
 * result is deterministic for a fixed rank count.  At the end dx is gathered
 * so every rank returns the full step (the reference's Engine::minimize_step
 * contract, engine.cpp:75-101).  Uniform 3x3 block systems only.
 *
 * The transport is one primitive: allgather of `count` doubles per rank into
 * nranks * count (rank-major).  YS NCCL transport: ncclAllGather on the
 * context stream (libnccl.so.2 is dlopen-ed, no link dependency).  Host
 * transport: a caller callback over HOST buffers (e.g. torch.distributed
 * gloo), used by the multi-process tests on one device.
 * ------------------------------------------------------------------------ */
typedef int (*ys_allgather_fn)(void* user, const double* send, double* recv, int64_t count);
/* ncclGetUniqueId; rank 0 creates it and the caller broadcasts the 128 bytes. */
int ys_dist_unique_id(unsigned char id[128]);
int ys_dist_init_nccl(ys_context* ctx, int32_t rank, int32_t nranks, const unsigned char id[128]);
int ys_dist_init_host(ys_context* ctx, int32_t rank, int32_t nranks, ys_allgather_fn fn, void* user);
/* Back to single-GPU solves (destroys the NCCL communicator). */
int ys_dist_finalize(ys_context* ctx);
/* The partition of the last distributed solve: bounds (nranks + 1 block-row
 * boundaries), this rank's halo rows received per iteration, export rows sent. */
int ys_dist_info(ys_context* ctx, int32_t* rank, int32_t* nranks, int64_t* bounds, int64_t* halo_rows,
                 int64_t* export_rows);
/* Owned-row evaluation of the distributed solve: the static stencil (SNH,
 * bending) instances this rank evaluates (those touching its rows; the
 * partition comes from the static structure) and the scene's total. */
int ys_dist_eval_counts(ys_context* ctx, int64_t* evaluated, int64_t* total);

/* Peer-memory transport (one NVSwitch node, <= 8 ranks): the same row
 * partition, owned-row evaluation and recurrence, but ONE persistent
 * cooperative kernel per rank runs the whole solve and exchanges through
 * NVLink peer memory with device-side flags (no host round trip or
 * collective launch per iteration): each rank stores the z of the rows its
 * peers need straight into their windows (they form their halo p = z + beta p
 * themselves), its partial sums into their value slots followed by a
 * release-store of the exchange's sequence number, and at the end its rows of
 * dx into every peer.  Partials are summed in rank order on every rank.
 * Replaces the reference's sharded spmv_add (solver.cpp:59-82) across GPUs.
 *
 * open: allocate this rank's window (after ys_finalize) and return its
 * cudaIpcMemHandle (64 bytes); connect: map every peer's window from the
 * rank-major table of nranks handles (the caller all-gathers them, e.g. over
 * torch.distributed).  ys_minimize_step then uses the peer-memory solve.
 * probe: without `seen`, release-store rank+1 into every peer's probe slot;
 * with `seen` (nranks values), read the slots the peers wrote (a mapping
 * test that needs no spinning kernel). */
int ys_dist_p2p_open(ys_context* ctx, int32_t rank, int32_t nranks, unsigned char handle[64]);
int ys_dist_p2p_connect(ys_context* ctx, const unsigned char* handles);
int ys_dist_p2p_probe(ys_context* ctx, int64_t* seen);
/* n contexts of ONE process on ONE device as the n ranks of the peer-memory
 * solve (the windows are plain device pointers), stepped together by
 * ys_dist_p2p_group_step: every rank's pre-solve work (owned-row evaluation,
 * assembly, preconditioner) in its own context, then one cooperative launch
 * running all ranks' views of the solve kernel — the emulation of a
 * multi-GPU job on one GPU (separate per-rank kernels that spin on each other
 * cannot share a device).  dx: n step buffers or NULL; stats: n records. */
int ys_dist_p2p_group(ys_context** ctxs, int32_t n);
int ys_dist_p2p_group_step(ys_context** ctxs, int32_t n, double tol, int64_t max_iter, double** dx,
                           ys_step_stats* stats);

/* ------------------------------------------------------------------------
 * Benchmark hooks: per-stage device times of the last minimize_step, measured
 * with CUDA events on the context's stream (ms): [0] refresh_dynamic,
 * [1] local eval, [2] assembly gather, [3] preconditioner build, [4] PCG,
 * [5] SpMV (sum over iterations), [6] total, [7] the peer-memory solve kernel of the
 * whole job (ys_dist_p2p_group_step); [8..11] persistent-PCG phase clocks,
 * [12..15] its sub-phase clocks (ms must hold 16 doubles).
 * counts[0] = kernel launches, counts[1] = indefinite 9x9 projections of the
 * last assembly, counts[2] = uniform-3x3 PCG path of the last solve (1 sliced-ELL
 * copy, 2 row gather from upper storage, 3 peer-memory distributed; 0 other), counts[3] = of the
 * indefinite projections, those done by the Jacobi fallback (counts must hold
 * 4 values).
 * ------------------------------------------------------------------------ */
int ys_set_profiling(ys_context* ctx, int32_t enabled);
int ys_stage_times(ys_context* ctx, double* ms, int64_t* counts);
/* Scene::bump_dynamic_epoch (scene.hpp:190): forces the next minimize_step
 * to rebuild the dynamic structure, as every refresh_dynamic_pairs does. */
int ys_bump_dynamic_epoch(ys_context* ctx);
/* The cudaStream_t every kernel of the context is launched on (for CUDA-event
 * timing by the caller). */
int ys_stream(ys_context* ctx, void** stream);
/* Execution options: "overlap" (default 1) evaluates the static energies on
 * side streams while minimize_step rebuilds the dynamic group; 0 runs the
 * stages sequentially (bitwise the same step).  "eval_evd" (default 1) projects
 * the indefinite 9x9 element Hessians by the clamped-eigenpair path
 * (tridiagonal QL + inverse iteration, verified; failures go to the Jacobi
 * EVD); 0 sends every element through the Jacobi EVD, 2 hands every element
 * to the fallback kernel (all within 1e-12 of the exact projection).
 * "pcg_copy" (default 1) solves uniform 3x3 systems over the sliced-ELL copy;
 * 0 takes the row-gather persistent kernel (the path used when the copy's
 * plan does not fit shared memory; tests). */
int ys_set_option(ys_context* ctx, const char* name, int64_t value);
/* Times one kernel class alone: reps launches bracketed by CUDA events on the
 * context stream.  which: 0 = SpMV row gather from upper storage (static +
 * dynamic), 1 = assembly gather + gradient / diagonal / preconditioner rows,
 * 2 = local evaluation of all energies, 3 = the PCG's SpMV through the
 * sliced-ELL copy (uniform 3x3 systems), 4 = FP64 FMA peak probe (bytes
 * returns its FLOPs per launch).  avg_ms per launch; bytes = algorithmic bytes
 * per launch. */
int ys_time_kernel(ys_context* ctx, int32_t which, int32_t reps, double* avg_ms, double* bytes);


#ifdef __cplusplus
}
#endif
#endif /* YASPS_B200_H */
