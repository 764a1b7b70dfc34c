// ys_context.cuh — host-side state of one engine context.
//
// Mirrors what relsim::Engine owns (engine.hpp:66-79): the gradient layout,
// the compiled static and dynamic energy groups, their BlockSparseHessian
// structures, the gradient and the diagonal accumulator — all device
// resident — plus the scene pieces the energies read (targets, point
// domains, unions, pair primitives).
#pragma once

#include <array>
#include <set>
#include <string>
#include <vector>

#include "ys_common.cuh"

namespace ys {

enum Kind : int32_t {
  K_SNH = 0,       // add_stable_neo_hookean (energies.cpp:49-118)
  K_BENDING = 1,   // add_bending (energies.cpp:129-155)
  K_INERTIA = 2,   // add_inertia (energies.cpp:168-174)
  K_ORTHO = 3,     // add_affine_orthogonality (energies.cpp:120-127)
  K_PP = 4,        // add_point_point_barrier (energies.cpp:30-47)
  K_REPULSIVE = 5, // add_repulsive_energy (energies.cpp:20-28)
  K_PT = 6,        // point-triangle barrier (not in the reference; ys_contact4.cuh)
  K_EE = 7,        // edge-edge barrier (not in the reference)
  K_PE = 8         // point-edge barrier (not in the reference)
};

const char* kind_name(int k);

struct Target {
  int64_t n = 0;
  int32_t rc = 0;
  int64_t start = 0;   // GradientLayout::boundaries[t]
  int64_t block0 = 0;  // first target-instance block
};

struct Domain {
  int32_t kind = 0;
  int64_t n = 0;
  int32_t ta = -1, tb = -1;
  std::vector<int64_t> h_v2b;
  std::vector<double> h_rest;  // affine rest / fixed positions
  DevBuf<int32_t> v2b;
  DevBuf<double> rest;
  int kappa() const { return kind == YS_POINTS_FREE ? 1 : kind == YS_POINTS_AFFINE ? 2 : 0; }
  int width() const { return kind == YS_POINTS_FREE ? 3 : kind == YS_POINTS_AFFINE ? 12 : 0; }
};

struct Union {
  std::vector<int32_t> children;
  int32_t kappa_u = 0, width = 0;
  DevBuf<DomainDev> d_child;
  DevBuf<int64_t> d_offsets;
  std::vector<int64_t> offsets() const;
};

// Candidate primitives of a contact stencil set (ys_stencil.cu): PT points x
// triangles, PE points x edges, EE edges x edges (self).
struct StencilPrims {
  int kind = 0;  // 0 none, K_PT, K_EE, K_PE
  bool self = false;
  int aa = 0, ab = 0;  // points per A / B primitive
  int64_t na = 0, nb = 0;
  DevBuf<int32_t> a, b;  // union indices
};

struct PairSet {
  int32_t uni = -1;
  int32_t arity = 2;  // points per instance: 2 (pairs), 3 (point-edge), 4 (point-triangle, edge-edge)
  bool dynamic = false;
  int64_t n = 0;
  std::vector<int64_t> h_pairs;
  bool host_stale = false;  // set by the device refresh; get_pairs downloads lazily
  DevBuf<int32_t> pairs;  // arity x n union-global indices
  StencilPrims prims;
};

// Device scratch of the contact-candidate refresh (ys_contact.cu), reused.
struct ContactScratch {
  DevBuf<double> pos;              // 3 x union size, union order
  DevBuf<double> part, boxes;
  DevBuf<uint64_t> keys, keys_out;  // per-child slices (B side of a child pair)
  DevBuf<int32_t> idx, idx_out;
  DevBuf<int32_t> cnt, off, scratch;
};

// A compiled energy term group (CompiledEnergy, assembly.hpp:75-103).
struct Energy {
  int32_t kind = 0;
  std::string name;
  bool dynamic = false;
  int32_t mode = YS_PROJECT_FULL;
  int64_t n = 0;  // instances
  int32_t kappa = 0, width = 0;
  double prm[6] = {0, 0, 0, 0, 0, 0};
  int32_t target = -1, domain = -1, pairset = -1;
  DevBuf<int32_t> conn;    // SNH/bending: 4 vertex ids per instance
  DevBuf<double> cdata;    // SNH: Binv(9)+vol; bending: l0; inertia: mass
  DevBuf<double> anchor;   // inertia: x_tilde (n x 3)
  std::vector<double> h_mass;

  // --- structure, rebuilt with the group
  DevBuf<DSlot> slots;     // n x kappa
  DevBuf<int32_t> m;       // compressed size per instance
  DevBuf<uint32_t> hoff, goff, doff, soff;  // per-instance exclusive offsets
  uint32_t hstride = 0, gstride = 0, dstride = 0, sstride = 0;  // uniform strides
  bool uniform = true;
  int64_t hbase = 0, gbase = 0, dbase = 0, sbase = 0;  // bases inside the group buffers
  int64_t hsize = 0, gsize = 0, ndest = 0, nslot = 0;
  std::set<int> compressed_sizes;
  bool built = false;
};

// BlockSparseHessian (assembly.hpp:19-60) of one group plus its assembly and
// SpMV plans.
struct Structure {
  std::vector<std::array<int64_t, 5>> groups;  // rows, cols, coord_start, count, value_start
  int64_t n_blocks = 0, n_values = 0;
  bool all33 = true;
  DevBuf<int32_t> row, col;     // per unique block (scalar coordinates)
  DevBuf<int8_t> br, bc;        // block shape per unique block
  DevBuf<int64_t> voff;         // value offset per unique block
  DevBuf<double> values;
  // H assembly plan: contributions sorted by key; segment k = block k.
  int64_t n_contrib = 0;
  DevBuf<int64_t> seg;          // n_blocks + 1
  DevBuf<uint32_t> perm;        // double offset of each sorted contribution
  DevBuf<double> hcontrib;
  // static gather order: per shape group, its unique blocks sorted by run
  // length (a warp's lanes then sum runs of similar length)
  std::vector<DevBuf<int32_t>> gorder;
  bool gorder_valid = false;
  // gradient plan: slot contributions sorted by gstart; segment per block row.
  int64_t n_gcontrib = 0;
  DevBuf<int32_t> gseg;         // NB + 1
  DevBuf<uint32_t> gperm;
  DevBuf<int32_t> glen;         // length of each sorted slot contribution
  DevBuf<double> gcontrib;
  DevBuf<int32_t> diag_uid;     // NB: unique block index of the (b,b) block, -1 if absent
  // SpMV plan: full (both triangle) row lists over block rows.
  DevBuf<int32_t> sp_rowptr;    // NB + 1
  DevBuf<int32_t> sp_ent;       // uid | (transposed << 31), row-sorted
  DevBuf<int32_t> sp_oth;       // first DoF of the other block side of entry j
  DevBuf<int32_t> sp_pos_n;     // per uid: position of its (r, c) entry
  DevBuf<int32_t> sp_pos_t;     // per uid: position of its transposed entry, -1 on the diagonal
  // 3x3 structures: upper-storage row plan (normal blocks are contiguous in u)
  DevBuf<int32_t> nrow;         // NB + 1: first unique block of each block row
  DevBuf<int32_t> trow;         // NB + 1: first transposed entry of each block row
  DevBuf<int2> tlist;           // (u, row DoF) of off-diagonal blocks, sorted by column block
  int32_t max_row_len = 0;
  uint64_t checksum = 0;
  bool checksum_valid = false;
};

struct PcgState {
  double gnorm, rz, php, alpha, beta, rel, tol, pad0;
  long long it, max_iter, hist_cap;
  int status;  // 0 running, 1 converged, 2 stagnated (pHp == 0), 3 curvature error, 4 residual error, 5 max_iter
  int fail_it;
  unsigned int counter1, counter2;
  unsigned long long phase_ns[4];  // persistent PCG: SpMV+pHp, reduce+update, reduce, p-update (CTA 0 view)
  unsigned long long aux_ns[4];    // kernel-specific sub-phase clocks (CTA 0 view)
};

// Row-partitioned multi-GPU solve (ys_dist.cu).  The plan is rebuilt per
// solve because the dynamic structure changes every Newton iteration.
struct Context;
constexpr int kMaxP2P = 8;  // ranks of the peer-memory solve (one NVSwitch node)

// Peer-memory transport (kind 3, ys_dist.cu): one device allocation per rank
// that the peers write into — exchange flags and values, the z rows the rank
// receives as halo, and the step rows of every rank.
struct P2PState {
  char* win = nullptr;      // this rank's window (cudaMalloc; IPC-exported)
  size_t win_bytes = 0;
  int64_t win_s = 0;        // DoFs the window was sized for
  void* peer[kMaxP2P] = {}; // peer windows (IPC-mapped, or the group's own windows)
  bool ipc[kMaxP2P] = {};   // peer[k] came from cudaIpcOpenMemHandle
  std::vector<Context*> group;  // emulated ranks of one process (all on one device), else empty
  unsigned long long solve_id = 0;     // identical on every rank: flags are (solve_id << 32 | exchange)
  DevBuf<uint32_t> mask;    // NB: ranks that need row R's z (bit k)
  DevBuf<uint8_t> hflag;
  DevBuf<int32_t> halo;     // rows owned elsewhere whose z this rank receives
  DevBuf<int32_t> nhalo;
  int64_t nhalo_host = 0;
  DevBuf<unsigned long long> bar;  // rank-local grid barrier counter
  int sm_share = 0;         // CTAs per rank of the last launch
};

struct DistState {
  int kind = 0;  // 0 off, 1 host callback transport, 2 NCCL, 3 peer memory (P2P)
  int rank = 0, nranks = 1;
  ys_allgather_fn fn = nullptr;
  void* user = nullptr;
  void* nccl = nullptr;               // ncclComm_t
  std::vector<int64_t> bounds;        // nranks + 1 block-row boundaries (last solve)
  std::vector<int64_t> exp_off;       // nranks + 1 offsets into the export list
  int64_t max_exp = 0, max_rows = 0;  // padded allgather sizes (rows)
  DevBuf<int64_t> dbounds, dexp_off;
  DevBuf<uint8_t> need;               // NB: row referenced across a rank boundary
  DevBuf<int32_t> exp;                // export rows of all ranks, sorted
  DevBuf<int32_t> nsel;
  DevBuf<double> send, recv, dsend, dall;
  std::vector<double> hsend, hrecv;   // host transport staging
  // Owned-row evaluation: the partition comes from the static structure (so
  // it is known before the step's evaluation and fixed across iterations);
  // each static stencil energy evaluates only the instances touching this
  // rank's rows (boundary instances on both sides).
  bool have_static = false;
  std::vector<int64_t> sbounds;               // nranks + 1 block-row boundaries
  std::vector<DevBuf<int32_t>> sel;           // per energy: selected instances (empty: all)
  std::vector<int64_t> nsel_e;                // per energy: count (-1: all)
  int64_t eval_owned = 0, eval_total = 0;     // static stencil instances evaluated / in the scene
  std::vector<DevBuf<int32_t>> gsel;          // per static shape group: unique blocks touching owned rows
  std::vector<int64_t> ngsel;
  P2PState p2p;
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int err_cls = 0;
  std::string version;

  std::vector<Target> targets;
  int64_t s = 0;
  bool finalized = false;
  std::vector<Domain> domains;
  std::vector<Union> unions;
  std::vector<PairSet> pairsets;
  std::vector<Energy> energies;
  uint64_t epoch = 0, seen_epoch = 0;

  // DoF state
  DevBuf<double> X, X0, G, DX;
  std::vector<std::vector<double>> h_target_init;

  // block rows (target instances)
  int64_t NB = 0, diag_vals = 0;
  bool uniform3 = true;
  DevBuf<int32_t> bstart, brc, dof2block;
  DevBuf<int64_t> bvoff;
  DevBuf<double> diag, minv;
  DevBuf<int32_t> bflag;  // preconditioner: 0 ok, 1 identity fallback, 2 regularized, 3 singular
  int32_t regularized = 0;

  Structure S[2];  // 0 static, 1 dynamic
  bool assembled = false, assembled_h = false;

  // PCG
  DevBuf<double> r, z, p, hp;
  DevBuf<PcgState> pcg;
  DevBuf<unsigned char> gridbar;
  DevBuf<double> partials;
  DevBuf<double> hist;
  int64_t hist_count = 0;
  int pcg_blocks = 0;
  cudaGraphExec_t pcg_exec = nullptr;
  cudaGraph_t pcg_graph = nullptr;
  bool pcg_cond = false;
  std::vector<uint64_t> pcg_key;
  DevBuf<double> scratch;
  DevBuf<int> errflag;
  DevBuf<int> flagsum;
  // EnergyDev arrays of batched small energies (k_eval_multi); one per call
  // that may run concurrently: [0] static / all, [1] dynamic, [2] odd static part
  DevBuf<unsigned char> multi_e[3];
  DevBuf<int64_t> multi_pre[3];  // [eval error flag, regularised blocks, first singular block]
  // sliced-ELL full copy of H_static + H_dynamic for the uniform 3x3 PCG (ys_sell.cuh)
  DevBuf<int32_t> sell_len, sell_col;
  DevBuf<int32_t> sell_perm, sell_lenq;  // position -> row (rows sorted by length per window), length by position
  DevBuf<int64_t> sell_soff;
  DevBuf<double> sell_val;
  DevBuf<int> sell_tw;  // max entry rows per warp (persistent PCG plan cache)
  int64_t sell_tw_nw = -1;  // grid (warps) sell_tw_host was computed for
  int sell_tw_host = 0;
  int sell_h = 0;
  bool sell_prepared = false;  // layout built by sell_prepare, values not yet filled
  bool sell_filled = false;    // values filled by sell_fill_early (the step's solve consumes them)
  int64_t sell_rows = 0, sell_slices = 0;  // entry rows, slices
  int64_t sell_r0 = 0, sell_r1 = 0;         // block-row range of the copy

  int pcg_path = 0;  // last uniform-3x3 solve: 1 sliced-ELL copy, 2 row gather (the copy's plan does not fit)

  // structure-build scratch (reused across dynamic rebuilds)
  DevBuf<unsigned char> cubtmp;
  DevBuf<uint64_t> k_in, k_out, ukey;
  DevBuf<uint32_t> p_in, gk_in, gk_out, gp_in;
  DevBuf<int32_t> flags, incl, ghead, heads;
  DevBuf<unsigned char> grpbuf;
  DevBuf<unsigned char> cnt4, ex4;   // per-instance counts / offsets of non-uniform energies
  DevBuf<unsigned char> summary;     // device-side structure summary
  void* pinned = nullptr;            // 64 KiB pinned staging for small D2H copies
  std::vector<int32_t> rc_classes;   // distinct target block sizes
  std::vector<DevBuf<int32_t>> rc_lists;  // block ids per rc class (non-uniform layouts)

  // two-pass projection of 9x9 edge-space Hessians (SNH, bending)
  DevBuf<double> evd_m;          // pending M (45 per entry)
  DevBuf<int32_t> evd_list;      // pending element ids
  DevBuf<unsigned int> evd_count;  // per energy: indefinite elements, then Jacobi-fallback elements
  DevBuf<int32_t> evd_fblist;      // fallback elements (local list positions)
  DevBuf<double> evd_scratch;      // pass-B reflector scratch (per thread, two streams)
  int64_t evd_last = 0;          // indefinite elements of the last assembly (diagnostics)

  // profiling
  bool profiling = false;
  bool overlap = true;  // static evaluation on side streams during the dynamic rebuild (ys_set_option)
  bool eval_low_priority = true;
  bool warned_pcg_fallback = false;
  int pcg_ctas = 0;  // CTAs per SM of the persistent uniform-3x3 PCG (0: the most that fit)  // the row-gather PCG fallback was announced
  int gather_wshift = 12;  // static gather order: run-length sort inside windows of 2^wshift blocks  // side stream of the static evaluation below the context stream's priority
  bool pcg_copy = true;  // uniform 3x3 solve over the sliced-ELL copy (false: the row-gather kernel; tests)
  int evd_mode = 1;     // pass-B projection: 1 clamped-eigenpair path + Jacobi fallback, 0 Jacobi only,
                       // 2 every element handed to the fallback list (tests)
  double stage_ms[8] = {0};
  double pcg_phase_ms[8] = {0};
  int64_t launches = 0;
  cudaEvent_t ev[10] = {};
  // second stream: the static energies' evaluation overlaps the dynamic rebuild
  cudaStream_t stream2 = nullptr;  // the static energies' evaluation and gather
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

  DistState dist;
  ContactScratch contact;

  // free-standing BSR systems (ys_bsr_*)
  struct Bsr {
    int64_t s = 0;
    Structure st;
    int64_t nb = 0;
    std::vector<int64_t> h_rows, h_cols;
  };
  std::vector<Bsr> bsrs;
};

// --- host entry points implemented across the .cu files --------------------
void ctx_finalize(Context& c);
void ctx_refresh_dynamic(Context& c, bool force);
void ctx_build_group(Context& c, int which);
void ctx_assemble(Context& c, bool project, bool with_hessian, int only = -1, cudaEvent_t join = nullptr,
                  bool check = true);
void ctx_eval_all(Context& c, bool project, bool with_hessian, int only = -1, cudaStream_t s = nullptr,
                  int part = -1, bool zero_counts = true);
void ctx_gather_all(Context& c, int only = -1, cudaStream_t s = nullptr);
double ctx_total_energy(Context& c, double* per_energy);
void ctx_apply_hessian_dev(Context& c, const double* x, double* y);
void ctx_build_preconditioner(Context& c);
void ctx_pcg(Context& c, double tol, int64_t max_iter, const double* g_dev, double* x_dev,
             ys_step_stats* stats);
void ctx_upload_domains(Context& c);
void ctx_dist_pcg(Context& c, double tol, int64_t max_iter, ys_step_stats* stats);
void ctx_dist_unique_id(unsigned char* id);
void ctx_dist_init_nccl(Context& c, int rank, int nranks, const unsigned char* id);
void ctx_dist_finalize(Context& c);
void ctx_dist_static_plan(Context& c);  // partition + owned-row instance lists (once)
void ctx_dist_p2p_open(Context& c, int rank, int nranks, unsigned char* handle);  // window + IPC handle
void ctx_dist_p2p_connect(Context& c, const unsigned char* handles);            // map the peers' windows
void ctx_dist_p2p_group(const std::vector<Context*>& cs);                       // emulated ranks, one device
void ctx_dist_p2p_solve(const std::vector<Context*>& cs, double tol, int64_t max_iter, ys_step_stats* stats);
void ctx_dist_p2p_probe(Context& c, int64_t* seen);
uint64_t structure_checksum(Context& c, Structure& st, int64_t total_dofs);
void ctx_refresh_pairs(Context& c, int pairset, double dhat, const int32_t* child_fixed,
                       int64_t* n_pairs);
void ctx_get_points(Context& c, int domain, double* out);
void ctx_refresh_stencils(Context& c, int set, double dhat, int64_t* n);  // ys_stencil.cu

// structure pieces reusable by the free-standing BSR path
void build_structure_from_keys(Context& c, Structure& st, DevBuf<uint64_t>& keys,
                               DevBuf<uint32_t>& payload, int64_t nkeys, int64_t total_dofs,
                               const BlocksDev& blocks, bool build_assembly_plan);
void build_spmv_plan(Context& c, Structure& st, const BlocksDev& blocks);
void spmv_structure(Context& c, Structure& st, const BlocksDev& blocks, const double* x, double* y,
                    bool accumulate, const PcgState* st_dev);

BlocksDev blocks_view(Context& c);
void drop_pcg_graph(Context& c);
void sell_build(Context& c, int lanes_per_row, int64_t r0 = 0, int64_t r1 = -1);  // ys_sell.cu
void sell_prepare(Context& c, int lanes_per_row, int64_t r0 = 0, int64_t r1 = -1);  // ys_sell.cu
void sell_fill_early(Context& c, cudaStream_t s);                                    // ys_sell.cu
void pcg_prepare(Context& c);  // ys_solver.cu
void spmv_sell(Context& c, const double* x, double* y);
int sell_max_warp_rows(Context& c, int64_t warps, int slices_per_warp);   // y = H x through the sliced-ELL copy
bool pcg_uses_conditional_graph(Context& c);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of SMs of the current device (grid sizing in multiples of the SM count).
int sm_count();

}  // namespace ys
