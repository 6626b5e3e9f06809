/*
 * hapt_b200.h -- C ABI of the B200-native HAPT planner hot path.
 *
 * The reference (meshpipe, arXiv 2509.24859 planner) exposes this path as
 * Python functions; the one native boundary it has is the Cython operator
 * `meshpipe._core.dp_sweep` (pkg/src/meshpipe/_core/_dp.pyx:14-97, selected in
 * _core/__init__.py:6-18).  This library replaces that operator and the work
 * around it with sm_100a kernels:
 *
 *   K1  hapt_tables_build      replaces ProfileStore._build + analytic_profile
 *                              (profiling.py:88-103, 212-286), boundary_costs
 *                              (profiling.py:128-147), DpTables.__init__
 *                              (planner.py:169-248) and feasible_t_values /
 *                              candidate_tmax (profiling.py:315-318,
 *                              planner.py:424-429).
 *   --  hapt_tables_finalize   the CSR/pool preparation used by the drop-in
 *                              dp_sweep path (tables handed in as arrays).
 *   K2  hapt_dp_sweep_batch    replaces _core.dp_sweep (_dp.pyx:48-95) called
 *                              once per t_max candidate by planner.dp_search
 *                              (planner.py:385-421) / batched_search
 *                              (planner.py:490-542): one call sweeps a whole
 *                              batch of candidates.
 *       hapt_dp_select         _extract_plan's best-s choice (planner.py:287-298)
 *                              per candidate + the sort_key merge
 *                              (planner.py:107-115, 535-541) as an argmin.
 *       hapt_dp_backtrack      _extract_plan's backpointer walk + K chain
 *                              (planner.py:300-338).
 *   K3  hapt_launch_counts     adaptive/classic/eager launch counts for many
 *                              plans (scheduling.py:69-124).
 *       hapt_sim_1f1b          makespan (+ optional node start times) of many
 *                              1F1B plans, equal to simulate(build_dag(...))
 *                              (simulation.py:73-149, 204-228).
 *       hapt_dag_longest_path  simulate() on an arbitrary (e.g. user-edited)
 *                              DAG in CSR form, with cycle detection
 *                              (simulation.py:204-228).
 *
 * Conventions: every pointer argument is DEVICE memory unless its name ends in
 * `_host`; no function allocates; the caller passes workspaces sized by the
 * matching *_bytes query.  `stream` is a cudaStream_t passed as void*.
 * Functions return HAPT_OK (0) or an HAPT_E* status; hapt_last_error() gives
 * the message (thread-local).  Infeasibility is data, as in the reference:
 * F = +inf, N = 0, bp = -1 (_dp.pyx:33-36).
 */
#ifndef HAPT_B200_H
#define HAPT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HAPT_OK = 0,
  HAPT_EINVAL = 1,     /* bad argument / unsupported shape                   */
  HAPT_ECUDA = 2,      /* CUDA runtime error                                  */
  HAPT_ENOSPACE = 3,   /* workspace too small                                 */
  HAPT_ECOMM = 4,      /* CommTooLargeError (scheduling.py:38-48, 116-117)    */
  HAPT_ESCHED = 5,     /* ScheduleError (scheduling.py:34, 102-113, 235-239)  */
  HAPT_ECHAIN = 6,     /* broken backpointer chain (planner.py:305-312)       */
  HAPT_ECYCLE = 7      /* CycleError: DAG not fully processed                 */
};

const char *hapt_last_error(void);
int hapt_version(void);
/* Kernels this library has enqueued since load (all entry points, all
   threads): the bench's gpu_launches evidence.  No reference counterpart. */
int64_t hapt_launches(void);

/* ------------------------------------------------------------------------ */
/* K1: cost tables                                                           */
/* ------------------------------------------------------------------------ */

/* Instance description (device pointers). Mirrors the inputs of
 * ProfileStore(layers, cluster, model, imbalance_ratio, dedup)
 * (profiling.py:173-197) and boundary_costs(layers, cluster). */
typedef struct {
  int32_t L;          /* layers                                              */
  int32_t n_meshes;
  int32_t n_opts;     /* sum over meshes of |enumerate_submeshes(mesh)|      */
  int32_t G;          /* total devices                                       */
  const double *layer_flops;    /* [L]   Layer.flops                          */
  const double *layer_params;   /* [L]   Layer.param_bytes                    */
  const double *layer_bbytes;   /* [L]   Layer.boundary_bytes                 */
  const int32_t *layer_sig;     /* [L]   id of Layer.signature (equal <=> equal) */
  const int32_t *mesh_hosts;    /* [n_meshes] DeviceMesh.hosts                */
  const int32_t *mesh_dph;      /* [n_meshes] devices_per_host                */
  const double *mesh_peak;      /* [n_meshes] peak_flops                      */
  const double *mesh_mem;       /* [n_meshes] mem_device                      */
  const double *mesh_intra_bw;  /* [n_meshes]                                 */
  const double *mesh_inter_bw;  /* [n_meshes]                                 */
  const double *cross_bw_next;  /* [n_meshes] bw(mesh m, mesh m+1); last unused */
  const int32_t *opt_n;         /* [n_opts] submesh hosts used (cluster.py:157-168 order) */
  const int32_t *opt_m;         /* [n_opts] devices per host used               */
  const int32_t *opt_mesh;      /* [n_opts] mesh index (options are mesh-major)  */
  const int32_t *ovr_index;     /* nullable [n_opts][L+2][L+2]: override row of a
                                   canonical entry, or -1 (apply_overrides,
                                   profiling.py:328-368)                       */
  const double *ovr_vals;       /* nullable [n_ovr][4] t_fwd,t_bwd,mem_params,mem_act */
  double cross_latency;
  double beta, efficiency, alpha, replication, act_factor; /* CostModel     */
  double imbalance_ratio;       /* rho (may be +inf)                          */
  double total_flops;           /* sum(l.flops) evaluated by the host (CPython
                                   3.12 sum() is compensated: keep it host-side) */
  double total_peak;            /* ClusterSpec.total_peak_flops, host-side    */
  int32_t dedup;
} hapt_model_desc;

/* One CSR entry of the feasible-span index, with everything the DP needs
 * about the transition (o,k)->i besides the layer state: 16 bytes, one
 * 128-bit broadcast load in the DP kernel. */
typedef struct {
  double tt;        /* t_tab[o,k,i]                                          */
  int32_t prank;    /* index of tt in the sorted t_max pool (tt <= t_max <=>
                       prank < #pool values <= t_max); INT32_MAX if tt is
                       not finite                                            */
  uint16_t i;       /* span end (1-based layer)                              */
  uint16_t kmax;    /* largest integer K with mp + K*ma <= cap (exact fp64),
                       saturated; the _dp.pyx:83 mask becomes kk <= kmax     */
} hapt_span;

/* Device tables (one instance). Carved out of ONE caller-owned buffer by
 * hapt_tables_init; filled by hapt_tables_build (K1) or, for the drop-in
 * dp_sweep path, by copying DpTables arrays in and calling
 * hapt_tables_finalize. Layouts are the reference DpTables layouts. */
typedef struct {
  int32_t L, G, n_opts, n_meshes, s_max, nnz_cap, pool_cap;
  double *t_tab, *mp_tab, *ma_tab;        /* [n_opts][L+2][L+2], +inf = infeasible */
  double *tf_raw, *tb_raw, *mp_raw, *ma_raw; /* profile incl. pruned cells  */
  int8_t *cell_state;   /* bit0 feasible, bit1 canonical, bits2-3 prune reason
                           (1 = oom, 2 = imbalance)                          */
  int32_t *canon_q;     /* [L+2][L+2] first span start with equal signature  */
  double *opt_cap;      /* [n_opts]                                          */
  int32_t *opt_mesh, *opt_devs, *opt_off;   /* [n_opts], [n_opts], [n_meshes+1] */
  double *cb_same, *cb_next;                /* [n_meshes][L+1]               */
  int32_t *g_mesh, *g_avail, *g_crow;       /* [G+1]; g_crow: boundary row used when
                                               g is the successor state (-1: none) */
  int32_t *span_off;    /* [n_opts*(L+2)+1]                                  */
  int32_t *span_items;  /* [nnz_cap]                                         */
  hapt_span *spans;     /* [nnz_cap]                                         */
  int32_t *span_srank;  /* [nnz_cap] min prank over this entry and the rest of
                           its row (non-decreasing along the row)            */
  uint16_t *row_kmin;   /* [n_opts*(L+2)] min kmax over the row: if it is >=
                           3s the memory mask cannot bind at layer s         */
  uint16_t *row_pos;    /* [n_opts*(L+2)][L+2] #row entries with span end <= i
                           (the layer-s scan of a row stops at i = L-s+1)    */
  double *pool;         /* [pool_cap] sorted unique feasible t (t_max candidates) */
  int64_t *counters;    /* [16]: 0 nnz, 1 pool_len, 2..7 StoreStats
                           (candidates, canonical, canonical_feasible, aliased,
                           pruned_oom, pruned_imbalance), 10 = 1 if the
                           remaining-device encoding is unsupported (below) */
  void *scratch;        /* internal                                          */
  size_t scratch_bytes;
} hapt_tables;

/* Bytes of the single buffer holding a hapt_tables for these dimensions. */
size_t hapt_tables_bytes(int32_t L, int32_t G, int32_t n_opts, int32_t n_meshes);
/* Point every member of *t into buf (device, >= hapt_tables_bytes). */
int hapt_tables_init(hapt_tables *t, void *buf, size_t buf_bytes, int32_t L,
                     int32_t G, int32_t n_opts, int32_t n_meshes);
/* K1: build every table from the description; counters are written on the
 * device (read them after synchronising `stream`). */
int hapt_tables_build(hapt_tables *t, const hapt_model_desc *desc, void *stream);
/* Given t_tab/mp_tab/ma_tab/opt_cap/opt_mesh/opt_devs/opt_off/cb_same/cb_next/
 * g_mesh/g_avail/span_off/span_items already in place, derive spans, span_ik,
 * g_crow, pool and counters[0..1]. s_max is taken from t->s_max.
 * Encoding requirement (checked on the device, counters[10] = 1 if violated;
 * the drop-in dp_sweep raises ValueError then): every option uses >= 1
 * device, g_mesh[1..G] names a mesh, and the boundary row a transition into
 * state g2 reads (cb_same[r] if g_mesh[g2] == r else cb_next[r], r the
 * caller's mesh, _dp.pyx:64-77) is the same for every caller of g2.
 * DpTables' encoding (planner.py:213-226, meshes consumed in order) always
 * satisfies it; the reference's Cython kernel accepts any encoding. */
int hapt_tables_finalize(hapt_tables *t, void *stream);

/* ------------------------------------------------------------------------ */
/* K2: stage-partition DP                                                    */
/* ------------------------------------------------------------------------ */

/* Optional outputs of a sweep; every member may be NULL.
 * F, N, bp_i, bp_o: the reference layout [n_cand][s_max+1][L+2][G+1]
 *   (dp_sweep's return tuple); the caller pre-fills F=+inf (F[c,0,L+1,0]=0),
 *   N=0, bp=-1; bp_i and bp_o must be given together.
 * bp_packed: [n_cand][s_max+1][L+2][G+1] int32 (o << 16) | i, written only
 *   for finite cells -- exactly the cells a backtrack visits -- so it needs
 *   no pre-fill; hapt_dp_walk reads it.
 * ntop: [n_cand][s_max+1] int32 N[s,1,G] (the DP launch bound of the first
 *   stage, checked by _extract_plan, planner.py:337-338). */
typedef struct {
  double *F;
  double *N;
  int32_t *bp_i;
  int32_t *bp_o;
  int32_t *bp_packed;
  int32_t *ntop;
} hapt_dp_full;

size_t hapt_dp_workspace_bytes(const hapt_tables *t, int32_t n_cand);
/* Sweep every candidate t_max in tmax[0..n_cand) through all s_max layers.
 * ftop [n_cand][s_max+1] receives F[s,1,G] (+inf when infeasible); states
 * [n_cand] receives the finite-cell count isfinite(F[1:]).sum()
 * (planner.py:418-420). full may be NULL. */
int hapt_dp_sweep_batch(const hapt_tables *t, const double *tmax, int32_t n_cand,
                        double *ftop, int64_t *states, const hapt_dp_full *full,
                        void *work, size_t work_bytes, void *stream);
/* hapt_dp_sweep_batch with the candidates per lane of the DP warps chosen
 * by the caller: cpl = 1, 2 or 4 (0 = the library's choice from the batch and
 * table sizes).  Results are identical for every choice; only speed differs.
 * A batch whose t_max values are spread over the pool (the search's
 * binary-search probes) runs fastest at 1: lanes with distant t_max share
 * one warp's bounds.  work_bytes = hapt_dp_workspace_bytes covers every cpl. */
int hapt_dp_sweep_batch_cpl(const hapt_tables *t, const double *tmax, int32_t n_cand,
                            double *ftop, int64_t *states, const hapt_dp_full *full,
                            void *work, size_t work_bytes, int32_t cpl, void *stream);

/* Per candidate: best_s = first s minimising F[s,1,G] + (B-1)*t_max over
 * finite entries, tstar = that total (+inf if none) (planner.py:287-298).
 * winner[0] = index of the lexicographic min (tstar, index) -- the sort_key
 * order, since t_max is unique and ascending in the pool (planner.py:107-115);
 * winner[0] = -1 when every candidate is infeasible. */
int hapt_dp_select(const double *ftop, const double *tmax, int32_t n_cand,
                   int32_t s_max, int64_t num_microbatches, double *tstar,
                   int32_t *best_s, int32_t *winner, void *stream);

/* The reference operator itself, one t_max: replaces _core.dp_sweep
 * (_dp.pyx:14-97) for a caller that keeps the reference's one-candidate loop.
 * F, N (fp64) and bp_i, bp_o (int32) are device arrays [s_max+1][L+2][G+1]
 * in the reference layout; the library writes every element (F = +inf but
 * F[0,L+1,0] = 0, N = 0, bp = -1, then the DP), so they need no pre-fill.
 * t_max <= 0 is HAPT_EINVAL (planner.py:396-397 raises). */
size_t hapt_dp_sweep_workspace_bytes(const hapt_tables *t);
int hapt_dp_sweep(const hapt_tables *t, double t_max, double *F, double *N, int32_t *bp_i,
                  int32_t *bp_o, void *work, size_t work_bytes, void *stream);

/* Re-sweep one candidate with backpointers and walk the chain from
 * (best_s, 1, G). stages [s_max][3] = (layer_start, layer_end, option);
 * kchain [s_max] = DP launch bounds K; n_stages [1]. */
size_t hapt_backtrack_workspace_bytes(const hapt_tables *t);
int hapt_dp_backtrack(const hapt_tables *t, double tmax, int32_t best_s,
                      int32_t *stages, int32_t *kchain, int32_t *n_stages,
                      void *work, size_t work_bytes, void *stream);

/* Backpointer walk (planner.py:300-312) over one candidate's packed
 * backpointers from a batch sweep (bp_cand = bp_packed + c * (s_max+1)(L+2)(G+1)):
 * stages [s_max][3] = (layer_start, layer_end, option), n_stages [1]
 * (-1: broken chain, -2: plan does not cover every layer and device). */
int hapt_dp_walk(const hapt_tables *t, const int32_t *bp_cand, int32_t best_s,
                 int32_t *stages, int32_t *n_stages, void *stream);

/* Number of DpTables entries with t <= t_max for each candidate: the
 * _activated_pairs batching key (planner.py:483-487). */
int hapt_activated_pairs(const hapt_tables *t, const double *tmax, int32_t n_cand,
                         int64_t *activated, void *stream);

/* ------------------------------------------------------------------------ */
/* K3: 1F1B schedule evaluation                                              */
/* ------------------------------------------------------------------------ */

enum { HAPT_COUNTS_CLASSIC = 0, HAPT_COUNTS_EAGER = 1, HAPT_COUNTS_ADAPTIVE = 2 };

/* Plans are packed: plan p owns stages [stage_off[p], stage_off[p+1]); its
 * boundary j (0-based) is comm[stage_off[p] + j], j < S_p - 1.
 * counts[stage_off[p] + i] = N_i. tmax may be NULL (slowest stage) or give a
 * per-plan override (adaptive_counts t_max argument). status[p] = HAPT_OK,
 * HAPT_ECOMM or HAPT_ESCHED. */
int hapt_launch_counts(int32_t n_plans, const int32_t *stage_off,
                       const double *t_fwd, const double *t_bwd,
                       const double *comm, const double *tmax, double epsilon,
                       int32_t kind, int32_t *counts, int32_t *status, void *stream);

/* makespan[p] of simulate(build_dag(t_fwd, t_bwd, comm, build_program(counts, B))).
 * num_mb [n_plans]. node_start/node_end (nullable) receive start/end times in
 * the reference node numbering (simulation.py:103-111) at node_off[p]
 * (int64 [n_plans]). ring_depth >= max_p N_1(p) + 1 sizes the per-link FIFOs
 * kept in `work` (hapt_sim_workspace_bytes). status[p]: HAPT_OK,
 * HAPT_ESCHED (B < N_1, bad counts) or HAPT_ECYCLE (program deadlocks). */
size_t hapt_sim_workspace_bytes(int64_t total_stages, int32_t ring_depth);
int hapt_sim_1f1b(int32_t n_plans, const int32_t *stage_off, const double *t_fwd,
                  const double *t_bwd, const double *comm, const int32_t *counts,
                  const int32_t *num_mb, double *makespan, double *node_start,
                  double *node_end, const int64_t *node_off, int32_t ring_depth,
                  int32_t *status, void *work, size_t work_bytes, void *stream);

/* Schedule reports of many traces: simulation.analyze(trace, mem_act) and
 * steady_state_rate(trace, stage=1) (simulation.py:310-395), from the node
 * times hapt_sim_1f1b wrote at node_off.  Per packed stage x of plan p
 * (stage s = x - stage_off[p]):
 *   stage_rep[6x .. 6x+5] = busy, window, bubble, bubble_fraction,
 *                           steady_bubble, peak_inflight_bytes
 *   peak_inflight[x]
 *   link_rep[3x .. 3x+2]  = fwd_time, bwd_time, overlap_ratio of boundary s
 *                           (NaN for the last stage)
 * steady_rate[p] = NaN where the reference raises SimulationError (fewer than
 * 4 aligned samples).  mem_act [total_stages] may be NULL (bytes 0).  status
 * (nullable) marks plans whose simulation failed: their rows are NaN / -1.
 * Every figure equals the reference's float bit for bit (CPython's
 * compensated sum() reproduced). */
int hapt_analyze_1f1b(int32_t n_plans, int32_t total_stages, const int32_t *stage_off,
                      const double *t_fwd, const double *t_bwd, const double *comm,
                      const int32_t *counts, const int32_t *num_mb, const double *mem_act,
                      const double *node_start, const double *node_end,
                      const int64_t *node_off, const int32_t *status, double *stage_rep,
                      int32_t *peak_inflight, double *link_rep, double *steady_rate,
                      void *stream);

/* The same two calls over a "trace" layout that a batched simulation writes
 * with whole-sector stores (the analysis path of PlanBatch.analyze): pairs
 * {start, end} of doubles, trace 16-byte aligned, plan p's pairs from pair
 * index trace_off[p] on (double index 2*trace_off[p]):
 *   stage s, op q of its 1F1B program (q in [0, 2B)):  pair 2sB + q
 *   link l, forward transfer of microbatch i:          pair 2SB + 2lB + i - 1
 *   link l, backward transfer of microbatch i:         pair 2SB + (2l+1)B + i - 1
 * B(4S - 2) pairs per plan (the reference's sink node is the makespan).
 * Figures equal hapt_sim_1f1b / hapt_analyze_1f1b's bit for bit. */
int hapt_sim_1f1b_trace(int32_t n_plans, const int32_t *stage_off, const double *t_fwd,
                        const double *t_bwd, const double *comm, const int32_t *counts,
                        const int32_t *num_mb, double *makespan, double *trace,
                        const int64_t *trace_off, int32_t ring_depth, int32_t *status,
                        void *work, size_t work_bytes, void *stream);
int hapt_analyze_1f1b_trace(int32_t n_plans, int32_t total_stages, const int32_t *stage_off,
                            const double *t_fwd, const double *t_bwd, const double *comm,
                            const int32_t *counts, const int32_t *num_mb,
                            const double *mem_act, const double *trace,
                            const int64_t *trace_off, const int32_t *status,
                            double *stage_rep, int32_t *peak_inflight, double *link_rep,
                            double *steady_rate, void *stream);

/* steady_state_rate(trace, stage) (simulation.py:374-395) of each plan at
 * its own stage rate_stage[p] (1-based; NULL = stage 1), from node times in
 * the reference numbering as hapt_sim_1f1b writes them (node_end unused).
 * NaN where the reference raises SimulationError or status[p] != 0. */
int hapt_steady_rate_1f1b(int32_t n_plans, const int32_t *stage_off, const int32_t *counts,
                          const int32_t *num_mb, const double *node_start,
                          const int64_t *node_off, const int32_t *rate_stage,
                          const int32_t *status, double *steady_rate, void *stream);

/* asap_tight (simulation.py:407-424) of a trace over a DAG given as successor
 * CSR: first_bad [1] = the smallest node v whose start is not
 * math.isclose(max over predecessors u of start[u] + duration[u], rel_tol,
 * abs_tol=1e-12) (or != 0 without predecessors); n_nodes if every node is
 * tight.  work >= hapt_asap_workspace_bytes(n_nodes). */
size_t hapt_asap_workspace_bytes(int32_t n_nodes);
int hapt_dag_asap_check(int32_t n_nodes, const int32_t *succ_off, const int32_t *succ_idx,
                        const int32_t *indeg, const double *duration, const double *start,
                        double rel_tol, int32_t *first_bad, void *work, size_t work_bytes,
                        void *stream);

/* Kernel timing for measurement (bench.py): while enabled, every DP sweep
 * launch is bracketed by CUDA events on its stream (and programmatic
 * dependent launch is off, so each interval is one kernel).  hapt_prof_read
 * synchronises, returns per kind (0 = dp_relax / dp_relax_compact, 1 =
 * dp_window, 2 = the rest of the sweep) the summed milliseconds and launch
 * counts since the last read, and resets. */
int hapt_prof_enable(int32_t on);
int hapt_prof_read(double *ms, int64_t *count, int32_t n_kinds);

/* Longest-path start times of an arbitrary DAG given as successor CSR:
 * start[v] = max_u (start[u] + duration[u]). processed [1] = number of nodes
 * reached (< n_nodes <=> cycle). */
size_t hapt_dag_workspace_bytes(int32_t n_nodes);
int hapt_dag_longest_path(int32_t n_nodes, const int32_t *succ_off,
                          const int32_t *succ_idx, const int32_t *indeg,
                          const double *duration, double *start, double *end,
                          double *makespan, int32_t *processed, void *work,
                          size_t work_bytes, void *stream);

/* ------------------------------------------------------------------------ */
/* Front end (host code)                                   */
/* ------------------------------------------------------------------------ */

/* detect_modules (model_graph.py:169-208): partition an operator sequence
 * into repeated / non-repeated modules.  tag_host [n_ops] = shape_tag ids
 * (equal tags <=> equal ids), heavy_host [n_ops] = 1 for HEAVY.  Outputs
 * (capacity n_ops) in position order: span start/end (half-open), group id
 * (-1 = non_repeated) and occurrence index.  Host memory. */
int hapt_detect_modules(int32_t n_ops, const int32_t *tag_host, const uint8_t *heavy_host,
                        int32_t z, int32_t *span_start_host, int32_t *span_end_host,
                        int32_t *span_group_host, int32_t *span_occ_host,
                        int32_t *n_spans_host);

/* cluster_layers (model_graph.py:269-333): u layers per module by min-max
 * flops partition (repeated groups share the first occurrence's cuts).
 * Outputs (capacity n_ops): op range, flops and param bytes (CPython 3.12
 * compensated sums, bit-identical), boundary bytes, signature triples
 * [kind (0 rep, 1 solo), group or solo ordinal, part].  Host memory. */
int hapt_cluster_layers(int32_t n_ops, const double *flops_host, const double *params_host,
                        const double *out_bytes_host, int32_t n_spans,
                        const int32_t *span_start_host, const int32_t *span_end_host,
                        const int32_t *span_group_host, int32_t u, int32_t *layer_start_host,
                        int32_t *layer_end_host, double *layer_flops_host,
                        double *layer_params_host, double *layer_bbytes_host,
                        int32_t *layer_sig_host, int32_t *n_layers_host);

/* CPython >= 3.12 sum() of n floats (Neumaier), for host-side aggregates. */
double hapt_py_sum(const double *x_host, int32_t n);

/* FP64 add-throughput probe (roofline denominator for K2/K3): runs `iters`
 * dependent-chain-free DADDs per thread; result[0] = checksum. */
int hapt_fp64_probe(double *result, int32_t blocks, int32_t threads,
                    int32_t iters, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HAPT_B200_H */
