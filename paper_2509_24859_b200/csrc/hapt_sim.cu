// K3 -- heterogeneity-aware 1F1B schedule evaluation, batched over plans.
//
// Reference path: adaptive_counts / classic_counts / eager_counts
// (scheduling.py:69-124) -> build_program (scheduling.py:230-252) ->
// build_dag (simulation.py:73-149) -> simulate (simulation.py:204-228).
//
// The reference materialises a DAG of B(4S-2)+1 nodes per plan and runs a
// Kahn sweep.  Start times are max-plus longest paths, and max is exact, so
// the result does not depend on the order in which a node's predecessors are
// visited.  hapt_sim_1f1b therefore never builds the DAG: one thread owns one
// plan and walks every stage's 1F1B program directly,
//     start = max(end of the previous op on the stage, dependency end)
// where the dependency of F[i,s] is the forward transfer CF[i,s-1] and of
// B[i,s] the backward transfer CB[i,s] (simulation.py:136-141); transfers
// serialise per link direction (simulation.py:130-133):
//     endCF[i,s] = max(endF[i,s], endCF[i-1,s]) + c_s
//     endCB[i,s] = max(endB[i,s+1], endCB[i-1,s]) + c_s.
// Transfer ends travel through per-link FIFOs (depth <= N_1 + 1, see
// DESIGN.md §K3).  Each node's end is the same single IEEE addition the
// reference performs (start[u] + duration[u]), so makespans and node times
// are bit-identical.
//
// hapt_dag_longest_path covers simulate() on DAGs that callers edited by hand
// (the reference tests corrupt one to provoke CycleError): a single-CTA
// frontier Kahn sweep with atomicMax on the (non-negative) double bit
// patterns.
#include <stdlib.h>

#include "hapt_common.cuh"

namespace hapt {
namespace {

constexpr int kMaxStages = 64;

__global__ void k_counts(int n_plans, const int32_t *stage_off, const double *t_fwd,
                         const double *t_bwd, const double *comm, const double *tmax,
                         double eps, int kind, int32_t *counts, int32_t *status) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_plans) return;
  const int b0 = stage_off[p], S = stage_off[p + 1] - b0;
  if (S < 1) {
    status[p] = HAPT_ESCHED;
    return;
  }
  double tm = 0.0;
  bool first = true;
  for (int i = 0; i < S; ++i) {
    const double t = __dadd_rn(t_fwd[b0 + i], t_bwd[b0 + i]);
    if (kind == HAPT_COUNTS_ADAPTIVE && !(t > 0.0)) {
      status[p] = HAPT_ESCHED;  // "stage times must be positive"
      return;
    }
    if (first || t > tm) tm = t;  // max(stage_times)
    first = false;
  }
  if (kind == HAPT_COUNTS_ADAPTIVE) {
    for (int i = 0; i + 1 < S; ++i)
      if (comm[b0 + i] < 0.0) {
        status[p] = HAPT_ESCHED;
        return;
      }
    if (tmax) {
      if (tmax[p] < tm) {
        status[p] = HAPT_ESCHED;  // "t_max override below the slowest stage time"
        return;
      }
      tm = tmax[p];
    }
  }
  int n = 1;
  counts[b0 + S - 1] = 1;
  for (int i = S - 2; i >= 0; --i) {
    int d;
    if (kind == HAPT_COUNTS_CLASSIC) {
      d = 1;
    } else if (kind == HAPT_COUNTS_EAGER) {
      d = 2;
    } else {
      const double c = comm[b0 + i];
      if (c > tm) {
        status[p] = HAPT_ECOMM;
        return;
      }
      if (c <= __dmul_rn(eps, tm)) d = 1;
      else if (c <= __ddiv_rn(tm, 2.0)) d = 2;
      else d = 3;
    }
    n += d;
    counts[b0 + i] = n;
  }
  status[p] = HAPT_OK;
}

// k-th op (0-based) of a stage with warm-up count N (scheduling.py:241-249):
// F1..FN | (B j, F N+j) for j = 1..B-N | B (B-N+1)..B.  Returns mb, sets isF.
__device__ __forceinline__ int decode_op(int pos, int N, int B, bool &isF) {
  if (pos < N) {
    isF = true;
    return pos + 1;
  }
  const int q = pos - N, steady = B - N;
  if (q < 2 * steady) {
    isF = (q & 1);
    return isF ? N + (q + 1) / 2 : q / 2 + 1;
  }
  isF = false;
  return steady + (q - 2 * steady) + 1;
}

// Inverse of decode_op: program position of (mb, F or B) on a stage.
__device__ __forceinline__ int encode_op(int mb, bool isF, int N, int B) {
  const int steady = B - N;
  if (isF) return mb <= N ? mb - 1 : N + 2 * (mb - N) - 1;
  return mb <= steady ? N + 2 * (mb - 1) : N + 2 * steady + (mb - steady - 1);
}

// Where a simulation puts per-node times (all pointers null: makespan only).
//   Reference numbering (simulation.py:103-111), start / end arrays: stage s
//     op (mb, F/B) at nb + 2(sB + mb - 1) + {0, 1}, link l transfer (mb,
//     fwd/bwd) at nb + 2SB + 2(lB + mb - 1) + {0, 1}, the sink last.
//   Trace layout, double2 {start, end}: stage s's ops in program order at
//     nb + 2sB + q, link l's forward transfers at nb + 2SB + 2lB + mb - 1 and
//     its backward ones B further on; no sink (it is the makespan).  A
//     thread writes each of its lists front to back, so every 32-byte sector
//     is complete after two consecutive stores instead of collecting four
//     scattered ones (partial sectors evicted from L2 cost a DRAM read).
// nb = off[p] in either layout.  Kernels that know the layout at compile
// time pass it as M (kRefNodes / kTrace); M = -1 decides at run time.
constexpr int kNoNodes = 0, kRefNodes = 1, kTrace = 2;

struct NodeOut {
  double *start, *end;
  double2 *trace;
  const int64_t *off;
  __host__ __device__ int mode() const {
    return trace ? kTrace : start ? kRefNodes : kNoNodes;
  }
  __device__ bool on() const { return start != nullptr || trace != nullptr; }
  template <int M = -1>
  __device__ void op(int64_t nb, int B, int s, int mb, bool isF, int q, double a,
                     double e) const {
    if (M < 0 ? trace != nullptr : M == kTrace) {
      trace[nb + 2 * (int64_t)s * B + q] = make_double2(a, e);
    } else {
      const int64_t id = nb + 2 * ((int64_t)s * B + (mb - 1)) + (isF ? 0 : 1);
      start[id] = a;
      end[id] = e;
    }
  }
  template <int M = -1>
  __device__ void xfer(int64_t nb, int S, int B, int l, int dir, int mb, double a,
                       double e) const {
    const int64_t base = nb + 2 * (int64_t)S * B + 2 * (int64_t)l * B;
    if (M < 0 ? trace != nullptr : M == kTrace) {
      trace[base + (int64_t)dir * B + (mb - 1)] = make_double2(a, e);
    } else {
      const int64_t id = base + 2 * (int64_t)(mb - 1) + dir;
      start[id] = a;
      end[id] = e;
    }
  }
  template <int M = -1>
  __device__ void sink(int64_t nb, int S, int B, double mk) const {
    if (M < 0 ? trace != nullptr : M == kTrace) return;
    const int64_t id = nb + 2 * (int64_t)S * B + 2 * (int64_t)(S - 1) * B;
    start[id] = mk;
    end[id] = mk;
  }
};

__global__ void k_sim(int n_plans, const int32_t *perm, const int32_t *n_perm,
                      const int32_t *stage_off, const double *t_fwd,
                      const double *t_bwd, const double *comm, const int32_t *counts,
                      const int32_t *num_mb, double *makespan, NodeOut out, int R,
                      double *ring, int32_t *status) {
  // all plans (perm == NULL) or the n_perm[0] plans listed in perm
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (perm ? *n_perm : n_plans)) return;
  const int p = perm ? perm[t] : t;
  const int b0 = stage_off[p], S = stage_off[p + 1] - b0, B = num_mb[p];
  if (S < 1 || S > kMaxStages || B < 1) {
    status[p] = HAPT_ESCHED;
    return;
  }
  // build_program preconditions (scheduling.py:235-239, 61-66)
  if (counts[b0 + S - 1] != 1 || B < counts[b0]) {
    status[p] = HAPT_ESCHED;
    return;
  }
  for (int s = 0; s < S; ++s)
    if (counts[b0 + s] < 1 || counts[b0 + s] > B || counts[b0 + s] + 1 > R) {
      status[p] = HAPT_ESCHED;
      return;
    }
  int pos[kMaxStages], fdone[kMaxStages], bdone[kMaxStages];
  double prev[kMaxStages], lcf[kMaxStages], lcb[kMaxStages];
  for (int s = 0; s < S; ++s) {
    pos[s] = fdone[s] = bdone[s] = 0;
    prev[s] = lcf[s] = lcb[s] = 0.0;
  }
  // FIFOs: link s forward at ring[(b0+s)*2R + slot], backward at +R
  double *rf = ring + (size_t)b0 * 2 * R;
  const bool want_nodes = out.on();
  const int64_t nb = want_nodes ? out.off[p] : 0;
  double mk = 0.0;
  int remaining = S;
  for (int s = 0; s < S; ++s) remaining -= (2 * B == 0);
  while (remaining > 0) {
    bool progress = false;
    for (int s = 0; s < S; ++s) {
      const int N = counts[b0 + s];
      while (pos[s] < 2 * B) {
        bool isF;
        const int mb = decode_op(pos[s], N, B, isF);
        double dep = 0.0;
        if (isF) {
          if (s > 0) {
            if (fdone[s - 1] < mb) break;
            dep = rf[(size_t)(s - 1) * 2 * R + (mb % R)];
          }
        } else {
          if (s < S - 1) {
            if (bdone[s + 1] < mb) break;
            dep = rf[(size_t)s * 2 * R + R + (mb % R)];
          }
        }
        const double st = fmax(prev[s], dep);
        const double d = isF ? t_fwd[b0 + s] : t_bwd[b0 + s];
        const double en = __dadd_rn(st, d);
        prev[s] = en;
        mk = fmax(mk, en);
        if (want_nodes) out.op(nb, B, s, mb, isF, pos[s], st, en);
        if (isF) {
          fdone[s] = mb;
          if (s < S - 1) {  // forward transfer on link s
            const double cs = fmax(en, lcf[s]);
            const double ce = __dadd_rn(cs, comm[b0 + s]);
            lcf[s] = ce;
            mk = fmax(mk, ce);
            rf[(size_t)s * 2 * R + (mb % R)] = ce;
            if (want_nodes) out.xfer(nb, S, B, s, 0, mb, cs, ce);
          }
        } else {
          bdone[s] = mb;
          if (s > 0) {  // backward transfer on link s-1
            const double cs = fmax(en, lcb[s - 1]);
            const double ce = __dadd_rn(cs, comm[b0 + s - 1]);
            lcb[s - 1] = ce;
            mk = fmax(mk, ce);
            rf[(size_t)(s - 1) * 2 * R + R + (mb % R)] = ce;
            if (want_nodes) out.xfer(nb, S, B, s - 1, 1, mb, cs, ce);
          }
        }
        ++pos[s];
        progress = true;
        if (pos[s] == 2 * B) --remaining;
      }
    }
    if (!progress) {
      status[p] = HAPT_ECYCLE;
      makespan[p] = kInf;
      return;
    }
  }
  if (want_nodes) out.sink(nb, S, B, mk);
  makespan[p] = mk;
  status[p] = HAPT_OK;
}

// General DAG: single-CTA frontier sweep (Kahn) -- simulation.py:204-228.
__global__ void k_dag(int n, const int32_t *succ_off, const int32_t *succ_idx,
                      const int32_t *indeg0, const double *dur, double *start, double *end,
                      double *makespan, int32_t *processed, int32_t *indeg, int32_t *fa,
                      int32_t *fb) {
  __shared__ int n_cur, n_next, n_done;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    indeg[v] = indeg0[v];
    start[v] = 0.0;
  }
  if (threadIdx.x == 0) {
    n_cur = 0;
    n_done = 0;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < n; v += blockDim.x)
    if (indeg0[v] == 0) fa[atomicAdd(&n_cur, 1)] = v;
  __syncthreads();
  int32_t *cur = fa, *nxt = fb;
  while (n_cur > 0) {
    if (threadIdx.x == 0) n_next = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < n_cur; j += blockDim.x) {
      const int u = cur[j];
      const double e = __dadd_rn(start[u], dur[u]);
      for (int x = succ_off[u]; x < succ_off[u + 1]; ++x) {
        const int v = succ_idx[x];
        atomicMax((unsigned long long *)&start[v], dkey(e));
      }
    }
    __syncthreads();  // all maxima in before any successor is released
    for (int j = threadIdx.x; j < n_cur; j += blockDim.x) {
      const int u = cur[j];
      for (int x = succ_off[u]; x < succ_off[u + 1]; ++x) {
        const int v = succ_idx[x];
        if (atomicSub(&indeg[v], 1) == 1) nxt[atomicAdd(&n_next, 1)] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      n_done += n_cur;
      n_cur = n_next;
    }
    int32_t *tmp = cur;
    cur = nxt;
    nxt = tmp;
    __syncthreads();
  }
  double mk = 0.0;
  for (int v = threadIdx.x; v < n; v += blockDim.x) {
    const double e = __dadd_rn(start[v], dur[v]);
    end[v] = e;
    mk = fmax(mk, e);
  }
  __shared__ double red[1024];
  red[threadIdx.x] = mk;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *makespan = red[0];
    *processed = n_done;
  }
}

// ---------------------------------------------------------------------------
// Fast path for plans with S <= 8 stages (config E): S is a template
// parameter, so every per-stage recurrence value (program position, last end
// on the stage, last transfer end per link direction, ops done) lives in
// registers; the per-link transfer FIFOs live in shared memory, [slot][thread]
// so a warp's accesses are conflict-free.  Stages advance round-robin, one op
// per sweep, which keeps the FIFOs shallow; a producer whose FIFO is full
// waits (max-plus results do not depend on the processing order).  A plan
// that stops progressing (a program that deadlocks, or FIFO capacity
// exceeded by unusual counts) is marked for the generic kernel.
// ---------------------------------------------------------------------------
#ifndef HAPT_SIM_RING
#define HAPT_SIM_RING 4
#endif
constexpr int kRing = HAPT_SIM_RING;  // FIFO slots per link direction (power of two)
constexpr int kRetry = -1;

template <int S>
struct SimCfg {
  static constexpr int threads = S >= 6 ? 64 : 128;
  static constexpr size_t smem = (size_t)(S > 1 ? S - 1 : 1) * 2 * kRing * threads * 8;
};

template <int S, int M>  // M: kNoNodes / kRefNodes / kTrace
__global__ void __launch_bounds__(SimCfg<S>::threads)
    k_sim_s(const int32_t *perm, int n, const int32_t *stage_off, const double *t_fwd,
            const double *t_bwd, const double *comm, const int32_t *counts,
            const int32_t *num_mb, double *makespan, int32_t *status, NodeOut out) {
  extern __shared__ double ring[];  // [(S-1) links][2 dirs][kRing][threads]
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int p = perm[t];
  const int b0 = stage_off[p], B = num_mb[p];
  int N[S];
  double tf[S], tb[S], cm[S > 1 ? S - 1 : 1];
  bool bad = B < 1;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    N[s] = counts[b0 + s];
    tf[s] = t_fwd[b0 + s];
    tb[s] = t_bwd[b0 + s];
    if (s + 1 < S) cm[s] = comm[b0 + s];
    bad |= N[s] < 1 || N[s] > B;
  }
  // build_program preconditions (scheduling.py:235-239, 61-66)
  if (bad || N[S - 1] != 1) {
    status[p] = HAPT_ESCHED;
    return;
  }
  const int ld = blockDim.x;
  auto slot = [&](int link, int dir, int mb) -> double & {
    return ring[(((link * 2 + dir) * kRing + (mb & (kRing - 1))) * ld) + threadIdx.x];
  };
  int pos[S], fd[S], bd[S];
  double prev[S], lcf[S], lcb[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    pos[s] = fd[s] = bd[s] = 0;
    prev[s] = lcf[s] = lcb[s] = 0.0;
  }
  double mk = 0.0;
  // optional per-node times in the reference numbering (simulation.py:103-111)
  constexpr bool nodes = M != kNoNodes;
  const int64_t nb = nodes ? out.off[p] : 0;
  int remaining = S;
  while (remaining > 0) {
    bool progress = false;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      if (pos[s] < 2 * B) {
        bool isF;
        const int mb = decode_op(pos[s], N[s], B, isF);
        bool ready;
        if (isF)
          ready = (s == 0 || fd[s - 1] >= mb) && (s == S - 1 || mb - fd[s + 1] <= kRing);
        else
          ready = (s == S - 1 || bd[s + 1] >= mb) && (s == 0 || mb - bd[s - 1] <= kRing);
        if (ready) {
          double dep = 0.0;
          if (isF && s > 0) dep = slot(s - 1, 0, mb);
          if (!isF && s < S - 1) dep = slot(s, 1, mb);
          const double st = fmax(prev[s], dep);
          const double en = __dadd_rn(st, isF ? tf[s] : tb[s]);
          prev[s] = en;
          mk = fmax(mk, en);
          if (nodes) out.op<M>(nb, B, s, mb, isF, pos[s], st, en);
          if (isF) {
            fd[s] = mb;
            if (s < S - 1) {  // forward transfer on link s (simulation.py:130-140)
              const double cs = fmax(en, lcf[s]);
              const double ce = __dadd_rn(cs, cm[s]);
              lcf[s] = ce;
              mk = fmax(mk, ce);
              slot(s, 0, mb) = ce;
              if (nodes) out.xfer<M>(nb, S, B, s, 0, mb, cs, ce);
            }
          } else {
            bd[s] = mb;
            if (s > 0) {  // backward transfer on link s-1
              const double cs = fmax(en, lcb[s - 1]);
              const double ce = __dadd_rn(cs, cm[s - 1]);
              lcb[s - 1] = ce;
              mk = fmax(mk, ce);
              slot(s - 1, 1, mb) = ce;
              if (nodes) out.xfer<M>(nb, S, B, s - 1, 1, mb, cs, ce);
            }
          }
          if (++pos[s] == 2 * B) --remaining;
          progress = true;
        }
      }
    }
    if (!progress) {
      status[p] = kRetry;  // let the generic kernel decide (deadlock vs. depth)
      return;
    }
  }
  if (nodes) out.sink<M>(nb, S, B, mk);
  makespan[p] = mk;
  status[p] = HAPT_OK;
}

// Makespan-only variant for 5-8 stages: one lane per stage, S consecutive
// lanes per plan (32 / S plans per warp).  Every round each lane tries the next op of its
// stage's program with the same readiness rules as k_sim_s (neighbours'
// progress read by shuffles at the start of the round, transfers through
// per-link FIFOs in shared memory, written in a round and read in a later
// one), so a plan advances up to S ops per round instead of one thread
// walking all S stages; the max-plus times are the same whatever the order.
// A plan none of whose lanes can move in a round is deadlocked or exceeds
// the FIFO depth and goes to the generic kernel, like k_sim_s's.
#ifndef HAPT_SIM_LANES_MIN
#define HAPT_SIM_LANES_MIN 7  // (S = 5, 6: k_sim_s measured faster -- 5.26 vs 5.10 ms per 10^6 config-E plans)
#endif
template <int S>
struct LaneCfg {
  static constexpr int per_warp = 32 / S;    // plans per warp
  static constexpr int plans = 4 * per_warp;  // plans per 128-thread block
};
template <int S, int M>  // M: kNoNodes / kRefNodes / kTrace, as k_sim_s
__global__ void __launch_bounds__(128)
    k_sim_l(const int32_t *perm, int n, const int32_t *stage_off, const double *t_fwd,
            const double *t_bwd, const double *comm, const int32_t *counts,
            const int32_t *num_mb, double *makespan, int32_t *status, NodeOut out) {
  constexpr int PW = LaneCfg<S>::per_warp;
  __shared__ double ring[LaneCfg<S>::plans][S > 1 ? S - 1 : 1][2][kRing];
  const int lane = threadIdx.x & 31;
  const int sub = lane / S, s = lane - sub * S, slot = (threadIdx.x >> 5) * PW + sub;
  const int t = blockIdx.x * LaneCfg<S>::plans + slot;
  const unsigned gmask = ((1u << S) - 1u) << (sub * S);
  const bool has = sub < PW && t < n;
  const int p = has ? perm[t] : 0;
  const bool act = has && s < S;
  const int b0 = has ? stage_off[p] : 0, B = has ? num_mb[p] : 1;
  int N = 1;
  double tf = 0.0, tb = 0.0, cmf = 0.0, cmb = 0.0;
  if (act) {
    N = counts[b0 + s];
    tf = t_fwd[b0 + s];
    tb = t_bwd[b0 + s];
    if (s + 1 < S) cmf = comm[b0 + s];
    if (s > 0) cmb = comm[b0 + s - 1];
  }
  // build_program preconditions (scheduling.py:235-239, 61-66)
  const bool bad = has && (B < 1 || (act && (N < 1 || N > B)) || (s == S - 1 && N != 1));
  const bool plan_bad = (__ballot_sync(0xffffffffu, bad) & gmask) != 0;
  if (plan_bad && s == 0) status[p] = HAPT_ESCHED;
  bool done = !act || plan_bad, stuck = false;
  int pos = 0, fd = 0, bd = 0;
  double prev = 0.0, lcf = 0.0, lcb = 0.0, mk = 0.0;
  double(*rg)[2][kRing] = ring[sub < PW ? slot : 0];
  constexpr bool nodes = M != kNoNodes;
  const int64_t nb = nodes && act ? out.off[p] : 0;
  for (;;) {
    const unsigned alive = __ballot_sync(0xffffffffu, !done);
    if (alive == 0u) break;
    const int fd_l = __shfl_up_sync(0xffffffffu, fd, 1), bd_l = __shfl_up_sync(0xffffffffu, bd, 1);
    const int fd_r = __shfl_down_sync(0xffffffffu, fd, 1);
    const int bd_r = __shfl_down_sync(0xffffffffu, bd, 1);
    bool ready = false, isF = false;
    int mb = 0;
    if (!done) {
      mb = decode_op(pos, N, B, isF);
      if (isF)
        ready = (s == 0 || fd_l >= mb) && (s == S - 1 || mb - fd_r <= kRing);
      else
        ready = (s == S - 1 || bd_r >= mb) && (s == 0 || mb - bd_l <= kRing);
    }
    if (ready) {
      double dep = 0.0;
      if (isF && s > 0) dep = rg[s - 1][0][mb & (kRing - 1)];
      if (!isF && s < S - 1) dep = rg[s][1][mb & (kRing - 1)];
      const double st = fmax(prev, dep);
      const double en = __dadd_rn(st, isF ? tf : tb);
      prev = en;
      mk = fmax(mk, en);
      if (nodes) out.op<M>(nb, B, s, mb, isF, pos, st, en);
      if (isF) {
        fd = mb;
        if (s < S - 1) {  // forward transfer on link s (simulation.py:130-140)
          const double cs = fmax(en, lcf);
          const double ce = __dadd_rn(cs, cmf);
          lcf = ce;
          mk = fmax(mk, ce);
          rg[s][0][mb & (kRing - 1)] = ce;
          if (nodes) out.xfer<M>(nb, S, B, s, 0, mb, cs, ce);
        }
      } else {
        bd = mb;
        if (s > 0) {  // backward transfer on link s-1
          const double cs = fmax(en, lcb);
          const double ce = __dadd_rn(cs, cmb);
          lcb = ce;
          mk = fmax(mk, ce);
          rg[s - 1][1][mb & (kRing - 1)] = ce;
          if (nodes) out.xfer<M>(nb, S, B, s - 1, 1, mb, cs, ce);
        }
      }
      if (++pos == 2 * B) done = true;
    }
    // a plan with live lanes none of which could move will never move
    const unsigned moved = __ballot_sync(0xffffffffu, ready);
    if ((alive & gmask) && !(moved & gmask)) {
      stuck = true;
      done = true;
    }
    __syncwarp();  // this round's FIFO writes before the next round's reads
  }
  // the plan's makespan: max over its lanes, gathered on its first lane
#pragma unroll
  for (int j = 1; j < S; ++j) {
    const double v = __shfl_down_sync(0xffffffffu, mk, j);
    if (s + j < S) mk = fmax(mk, v);
  }
  if (has && s == 0 && !plan_bad) {
    if (stuck) {
      status[p] = kRetry;
    } else {
      if (nodes) out.sink<M>(nb, S, B, mk);
      makespan[p] = mk;
      status[p] = HAPT_OK;
    }
  }
}

// Counting sort of plan indices by stage count (bucket S for 1..8, bucket 0
// for S > 8): per-block histograms, one scan, per-block scatter.  Order inside
// a bucket is irrelevant (plans are independent).
constexpr int kBucketBlock = 1024;

__device__ __forceinline__ int bucket_of(const int32_t *stage_off, int p) {
  const int S = stage_off[p + 1] - stage_off[p];
  return (S >= 1 && S <= 8) ? S : 0;
}

__global__ void k_bucket_hist(int n_plans, const int32_t *stage_off, int32_t *bhist) {
  __shared__ int c[9];
  if (threadIdx.x < 9) c[threadIdx.x] = 0;
  __syncthreads();
  const int p = blockIdx.x * kBucketBlock + threadIdx.x;
  if (p < n_plans) atomicAdd(&c[bucket_of(stage_off, p)], 1);
  __syncthreads();
  if (threadIdx.x < 9) bhist[blockIdx.x * 9 + threadIdx.x] = c[threadIdx.x];
}

__global__ void k_bucket_scan(int n_blocks, int32_t *bhist, int32_t *cnt) {
  // one thread per bucket: exclusive scan over blocks, then bucket bases
  __shared__ int tot[9];
  const int b = threadIdx.x;
  if (b < 9) {
    int run = 0;
    for (int k = 0; k < n_blocks; ++k) {
      const int v = bhist[k * 9 + b];
      bhist[k * 9 + b] = run;
      run += v;
    }
    tot[b] = run;
    cnt[b] = run;
  }
  __syncthreads();
  if (b < 9) {
    int base = 0;
    for (int q = 0; q < b; ++q) base += tot[q];
    cnt[10 + b] = base;  // bucket start in perm
  }
}

__global__ void k_bucket_scatter(int n_plans, const int32_t *stage_off, const int32_t *bhist,
                                 const int32_t *cnt, int32_t *perm) {
  __shared__ int c[9];
  if (threadIdx.x < 9) c[threadIdx.x] = 0;
  __syncthreads();
  const int p = blockIdx.x * kBucketBlock + threadIdx.x;
  if (p < n_plans) {
    const int b = bucket_of(stage_off, p);
    perm[cnt[10 + b] + bhist[blockIdx.x * 9 + b] + atomicAdd(&c[b], 1)] = p;
  }
}

__global__ void k_sim_retry(int n_plans, const int32_t *status, int32_t *perm, int32_t *n_out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_plans && status[p] == kRetry) perm[atomicAdd(n_out, 1)] = p;
}

template <int S>
void launch_sim_s(const int32_t *perm, int n, const int32_t *stage_off, const double *t_fwd,
                  const double *t_bwd, const double *comm, const int32_t *counts,
                  const int32_t *num_mb, double *makespan, int32_t *status, NodeOut out,
                  cudaStream_t st) {
  if (n <= 0) return;
  using C = SimCfg<S>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sim_s<S, kNoNodes>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::smem);
    cudaFuncSetAttribute(k_sim_s<S, kRefNodes>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::smem);
    cudaFuncSetAttribute(k_sim_s<S, kTrace>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::smem);
    attr = true;
  }
  const unsigned grid = grid_for(n, C::threads);
  const int m = out.mode();
  static const bool lanes = [] {
    const char *e = getenv("HAPT_SIM_LANES");
    return !(e && e[0] == '0');
  }();
  if constexpr (S >= HAPT_SIM_LANES_MIN && S <= 8) {
    if (lanes) {
      const unsigned lg = grid_for(n, LaneCfg<S>::plans);
      if (m == kTrace)
        k_sim_l<S, kTrace><<<lg, 128, 0, st>>>(perm, n, stage_off, t_fwd, t_bwd, comm, counts,
                                               num_mb, makespan, status, out);
      else if (m == kRefNodes)
        k_sim_l<S, kRefNodes><<<lg, 128, 0, st>>>(perm, n, stage_off, t_fwd, t_bwd, comm, counts,
                                                  num_mb, makespan, status, out);
      else
        k_sim_l<S, kNoNodes><<<lg, 128, 0, st>>>(perm, n, stage_off, t_fwd, t_bwd, comm, counts,
                                                 num_mb, makespan, status, out);
      ::hapt::note_launch();
      return;
    }
  }
  if (m == kTrace)
    k_sim_s<S, kTrace><<<grid, C::threads, C::smem, st>>>(
        perm, n, stage_off, t_fwd, t_bwd, comm, counts, num_mb, makespan, status, out);
  else if (m == kRefNodes)
    k_sim_s<S, kRefNodes><<<grid, C::threads, C::smem, st>>>(
        perm, n, stage_off, t_fwd, t_bwd, comm, counts, num_mb, makespan, status, out);
  else
    k_sim_s<S, kNoNodes><<<grid, C::threads, C::smem, st>>>(
        perm, n, stage_off, t_fwd, t_bwd, comm, counts, num_mb, makespan, status, out);
  ::hapt::note_launch();
}

// ---------------------------------------------------------------------------
// Schedule analysis (simulation.analyze / steady_state_rate, simulation.py:
// 310-395) over the node times of many traces.  Every reduction is a CPython
// builtin sum() over floats -- Neumaier-compensated since 3.12 -- and every
// interval list is produced in the order the reference's sorted()-based
// helpers see it, so each figure is the reference's float bit for bit.
// ---------------------------------------------------------------------------

// sum() of a float sequence: int 0 + first item, then Neumaier (bltinmodule.c)
struct PySum {
  double f = 0.0, c = 0.0;
  bool any = false;
  __device__ void add(double x) {
    if (!any) {
      f = __dadd_rn(0.0, x);
      any = true;
      return;
    }
    const double t = __dadd_rn(f, x);
    if (fabs(f) >= fabs(x))
      c = __dadd_rn(c, __dadd_rn(__dadd_rn(f, -t), x));
    else
      c = __dadd_rn(c, __dadd_rn(__dadd_rn(x, -t), f));
    f = t;
  }
  __device__ double value() const {
    return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f;
  }
};

// Sweep-line cursor over one serial interval list: a stage's ops in program
// order (start = max(previous end, dependency) >= previous end) or one link
// direction's transfers in microbatch order (endCF[i] = max(endF[i],
// endCF[i-1]) + c, so each starts after the previous one ends).  The list's
// boundaries lo0 <= hi0 <= lo1 <= hi1 <= ... are visited in order; empty
// intervals (hi <= lo) are skipped, as _interval_union drops them.
template <class At>
struct Serial {
  At at;               // interval k -> {lo, hi}
  int n, k;            // intervals, next interval to open
  bool open;           // inside interval k-1
  double x, hi;        // next boundary; end of the open interval
  __device__ void load() {  // x = start of the next non-empty interval
    for (; k < n; ++k) {
      const double2 v = at(k);
      hi = v.y;
      if (v.y > v.x) {
        x = v.x;
        ++k;
        return;
      }
    }
    x = kInf;
  }
  __device__ void init() {
    k = 0;
    open = false;
    load();
  }
  __device__ void step(double c) {  // apply every boundary at coordinate c
    while (x == c) {
      if (open) {
        open = false;
        load();
      } else {
        open = true;
        x = hi;
      }
    }
  }
};

// Node times as a simulation wrote them (NodeOut's two layouts).
struct NodeIn {
  const double *start, *end;
  const double2 *trace;
  const int64_t *off;
};

template <bool TRACE>
struct StageAt {  // op q of a stage in program order -> {start, end}
  NodeIn in;
  int64_t base;   // nb + 2sB
  int N, B;
  __device__ double2 operator()(int q) const {
    if constexpr (TRACE) {
      return __ldg(in.trace + base + q);
    } else {
      bool isF;
      const int mb = decode_op(q, N, B, isF);
      const int64_t id = base + 2 * (int64_t)(mb - 1) + (isF ? 0 : 1);
      return make_double2(in.start[id], in.end[id]);
    }
  }
};

template <bool TRACE>
struct LinkAt {  // transfer of microbatch i+1 in one direction -> {start, end}
  NodeIn in;
  int64_t base;   // nb + 2SB + 2lB
  int dir, B;     // 0 forward, 1 backward
  __device__ double2 operator()(int i) const {
    if constexpr (TRACE) {
      return __ldg(in.trace + base + (int64_t)dir * B + i);
    } else {
      const int64_t id = base + 2 * (int64_t)i + dir;
      return make_double2(in.start[id], in.end[id]);
    }
  }
};

// steady_state_rate(trace, stage) (simulation.py:374-395): least-squares
// slope of the forward start times of microbatches 2K+1, 3K+1, ... <= B on
// stage s0 (0-based), K its launch count; NaN where the reference raises
// SimulationError (fewer than 4 samples).  Sums are CPython's compensated
// sum(), the mean/deviation expressions the reference's.
template <bool TRACE>
__device__ double steady_rate_at(const NodeIn &in, int64_t nb, int s0, int K, int B) {
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  int n = 0;
  long long sx = 0;
  for (int i = 2 * K + 1; i <= B; i += K) ++n, sx += i;
  if (n < 4) return nan;
  const double fn = (double)n;
  const double mx = __ddiv_rn((double)sx, fn);
  PySum sy;
  // start of F(mb i) on stage s0
  const StageAt<TRACE> at0{in, nb + 2 * (int64_t)s0 * B, K, B};
  auto f_start = [&](int i) { return at0(encode_op(i, true, K, B)).x; };
  for (int i = 2 * K + 1; i <= B; i += K) sy.add(f_start(i));
  const double my = __ddiv_rn(sy.value(), fn);
  PySum sxx, sxy;
  for (int i = 2 * K + 1; i <= B; i += K) {
    const double dx = __dadd_rn((double)i, -mx);
    sxx.add(__dmul_rn(dx, dx));  // (x - mean_x) ** 2
    sxy.add(__dmul_rn(dx, __dadd_rn(f_start(i), -my)));
  }
  return __ddiv_rn(sxy.value(), sxx.value());
}

// steady_state_rate of plan p at its stage rate_stage[p] (1-based), node
// times in the reference numbering (simulate's trace).
__global__ void k_steady_rate(int n_plans, const int32_t *stage_off, const int32_t *counts,
                              const int32_t *num_mb, NodeIn in, const int32_t *rate_stage,
                              const int32_t *status, double *steady_rate) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_plans) return;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const int S = stage_off[p + 1] - stage_off[p];
  const int st = rate_stage ? rate_stage[p] : 1;
  if ((status && status[p] != HAPT_OK) || st < 1 || st > S) {
    steady_rate[p] = nan;
    return;
  }
  steady_rate[p] =
      steady_rate_at<false>(in, in.off[p], st - 1, counts[stage_off[p] + st - 1], num_mb[p]);
}

// asap_tight (simulation.py:407-424): every node with predecessors starts at
// max over them of start[u] + duration[u] (math.isclose(rel_tol, abs 1e-12)),
// every other node at 0.  Pass 1 (per node u, over its successors): the max
// as an order-preserving key; pass 2 (per node): the check, first failing
// node into *bad (n if none).
__device__ __forceinline__ unsigned long long okey(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_decode(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__global__ void k_asap_max(int n, const int32_t *succ_off, const int32_t *succ_idx,
                           const double *dur, const double *start, unsigned long long *hi) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const unsigned long long e = okey(__dadd_rn(start[u], dur[u]));
  for (int x = succ_off[u]; x < succ_off[u + 1]; ++x) atomicMax(hi + succ_idx[x], e);
}
// CPython math.isclose(a, b, rel_tol, abs_tol)
__device__ __forceinline__ bool py_isclose(double a, double b, double rel, double abs_tol) {
  if (a == b) return true;
  if (isinf(a) || isinf(b)) return false;
  const double diff = fabs(__dadd_rn(b, -a));
  return diff <= fabs(__dmul_rn(rel, b)) || diff <= fabs(__dmul_rn(rel, a)) || diff <= abs_tol;
}
__global__ void k_asap_check(int n, const int32_t *indeg, const double *start,
                             const unsigned long long *hi, double rel_tol, int32_t *bad) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const bool ok = indeg[v] == 0 ? start[v] == 0.0
                                : py_isclose(start[v], okey_decode(hi[v]), rel_tol, 1e-12);
  if (!ok) atomicMin(bad, v);
}

// Three thread ranges, so that a warp's threads run the same kind of row
// (a mixed warp serialises a long link walk behind short stage rows):
//   [0, T)        the stage row of packed stage x
//   [T, 2T)       the link row behind packed stage x (NaN on a plan's last stage)
//   [2T, 2T + P)  steady_state_rate of plan p
// (T = total stages, P = plans; plan p owns stages [stage_off[p], stage_off[p+1])).
template <bool TRACE>
__global__ void k_analyze(int n_plans, const int32_t *stage_off, const double *t_fwd,
                          const double *t_bwd, const double *comm, const int32_t *counts,
                          const int32_t *num_mb, const double *mem_act, NodeIn in,
                          const int32_t *status, double *stage_rep,
                          int32_t *peak_inflight, double *link_rep, double *steady_rate) {
  const long T = stage_off[n_plans];
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int role = t < T ? 0 : t < 2 * T ? 1 : t < 2 * T + n_plans ? 2 : 3;
  if (role == 3) return;
  int p, x;
  if (role == 2) {
    p = (int)(t - 2 * T);
    x = stage_off[p];
  } else {
    x = (int)(role == 0 ? t : t - T);
    int lo = 0, hi = n_plans;  // plan p: stage_off[p] <= x < stage_off[p+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (stage_off[mid] <= x) lo = mid; else hi = mid;
    }
    p = lo;
  }
  const int b0 = stage_off[p], S = stage_off[p + 1] - b0, s = x - b0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const bool failed = status && status[p] != HAPT_OK;
  const int B = num_mb[p];
  const int64_t nb = in.off[p];
  if (role == 0) {  // -- stage row (simulation.py:331-358) --
    if (failed) {
      for (int q = 0; q < 6; ++q) stage_rep[(size_t)x * 6 + q] = nan;
      peak_inflight[x] = -1;
      return;
    }
    const int N = counts[x];
    const int64_t base = nb + 2 * (int64_t)s * B;
    PySum busy, steady;
    int inflight = 0, peak = 0;
    const int w0 = N, w1 = N + 2 * (B - N);  // steady ops [w0, w1)
    for (int q = 0; q < 2 * B; ++q) {
      bool isF;
      decode_op(q, N, B, isF);
      const double d = isF ? t_fwd[x] : t_bwd[x];
      busy.add(d);
      if (q >= w0 && q < w1) steady.add(d);
      inflight += isF ? 1 : -1;
      peak = inflight > peak ? inflight : peak;
    }
    const StageAt<TRACE> at{in, base, N, B};
    const double first_start = at(0).x, last_end = at(2 * B - 1).y;
    const double steady_start = w1 > w0 ? at(w0).x : 0.0;
    const double steady_end = w1 > w0 ? at(w1 - 1).y : 0.0;
    const double bs = busy.value();
    const double window = __dadd_rn(last_end, -first_start);
    const double bubble = __dadd_rn(window, -bs);
    const double sb = w1 > w0 ? __dadd_rn(__dadd_rn(steady_end, -steady_start), -steady.value())
                              : 0.0;
    double *r = stage_rep + (size_t)x * 6;
    r[0] = bs;
    r[1] = window;
    r[2] = bubble;
    r[3] = window > 0.0 ? __ddiv_rn(bubble, window) : 0.0;
    r[4] = sb;
    r[5] = __dmul_rn((double)peak, mem_act ? mem_act[x] : 0.0);
    peak_inflight[x] = peak;
    return;
  }
  if (role == 1) {  // -- link row for boundary s (simulation.py:360-378) --
    double *lr = link_rep + (size_t)x * 3;
    if (failed || s >= S - 1) {
      lr[0] = lr[1] = lr[2] = nan;
      return;
    }
    const double c = comm[x];
    PySum f;
    for (int q = 0; q < B; ++q) f.add(c);
    const double ft = f.value();
    // One sweep over the four serial lists.  busy = _interval_union(forward
    // + backward transfers) is where either direction is open; its pieces are
    // the maximal runs of that (touching transfers merge: all boundaries at a
    // coordinate apply before the state is read).  _intersect(_intersect(busy,
    // stage s), stage s+1) yields exactly the maximal runs where busy and both
    // stages are open, each as [max of starts, min of ends] — the boundary
    // coordinates here — in increasing order, so both sums see the
    // reference's terms in the reference's order.
    const int64_t lbase = nb + 2 * (int64_t)S * B + 2 * (int64_t)s * B;
    Serial<LinkAt<TRACE>> cf{LinkAt<TRACE>{in, lbase, 0, B}, B};
    Serial<LinkAt<TRACE>> cb{LinkAt<TRACE>{in, lbase, 1, B}, B};
    Serial<StageAt<TRACE>> u0{StageAt<TRACE>{in, nb + 2 * (int64_t)s * B, counts[x], B}, 2 * B};
    Serial<StageAt<TRACE>> u1{
        StageAt<TRACE>{in, nb + 2 * (int64_t)(s + 1) * B, counts[x + 1], B}, 2 * B};
    cf.init();
    cb.init();
    u0.init();
    u1.init();
    PySum tot, both;
    bool in_busy = false, in_all = false;
    double busy0 = 0, all0 = 0;
    while (cf.x < kInf || cb.x < kInf) {  // no pieces outside busy
      const double at = fmin(fmin(cf.x, cb.x), fmin(u0.x, u1.x));
      cf.step(at);
      cb.step(at);
      u0.step(at);
      u1.step(at);
      const bool b = cf.open || cb.open;
      const bool a = b && u0.open && u1.open;
      if (a != in_all) {
        if (a) all0 = at; else both.add(__dadd_rn(at, -all0));
        in_all = a;
      }
      if (b != in_busy) {
        if (b) busy0 = at; else tot.add(__dadd_rn(at, -busy0));
        in_busy = b;
      }
    }
    const double total = tot.any ? tot.value() : 0.0;
    const double ratio =
        total > 0.0 ? __ddiv_rn(both.any ? both.value() : 0.0, total) : 1.0;
    lr[0] = ft;
    lr[1] = ft;  // backward transfers carry the same boundary time
    lr[2] = ratio;
    return;
  }
  // -- steady_state_rate(trace, stage=1) (simulation.py:374-395) --
  steady_rate[p] = failed ? nan : steady_rate_at<TRACE>(in, nb, 0, counts[x], B);
}

}  // namespace
}  // namespace hapt

using namespace hapt;

extern "C" int hapt_launch_counts(int32_t n_plans, const int32_t *stage_off, const double *t_fwd,
                                  const double *t_bwd, const double *comm, const double *tmax,
                                  double epsilon, int32_t kind, int32_t *counts, int32_t *status,
                                  void *stream) {
  if (n_plans < 1 || !stage_off || !t_fwd || !t_bwd || !comm || !counts || !status ||
      kind < 0 || kind > 2) {
    set_error("hapt_launch_counts: invalid arguments");
    return HAPT_EINVAL;
  }
  k_counts<<<grid_for(n_plans, 128), 128, 0, (cudaStream_t)stream>>>(
      n_plans, stage_off, t_fwd, t_bwd, comm, tmax, epsilon, kind, counts, status); ::hapt::note_launch();
  HAPT_LAUNCHED("k_counts");
  return HAPT_OK;
}

namespace {
// tail of the workspace: plan permutation, bucket counters, block histograms
size_t sim_tail_bytes(size_t n_plans) {
  return align_up(n_plans * 4) + align_up(32 * 4) +
         align_up((n_plans / kBucketBlock + 1) * 9 * 4);
}
}  // namespace

extern "C" size_t hapt_sim_workspace_bytes(int64_t total_stages, int32_t ring_depth) {
  const size_t ts = (size_t)(total_stages > 0 ? total_stages : 1);
  // generic-kernel FIFOs + tail sized for n_plans <= total_stages
  return align_up(ts * 2 * ring_depth * 8) + sim_tail_bytes(ts);
}

namespace {
int sim_1f1b(const char *who, int32_t n_plans, const int32_t *stage_off, const double *t_fwd,
             const double *t_bwd, const double *comm, const int32_t *counts,
             const int32_t *num_mb, double *makespan, NodeOut out, int32_t ring_depth,
             int32_t *status, void *work, size_t work_bytes, void *stream) {
  if (n_plans < 1 || !stage_off || !t_fwd || !t_bwd || !comm || !counts || !num_mb ||
      !makespan || !status || !work || ring_depth < 2) {
    set_error("%s: invalid arguments", who);
    return HAPT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const bool nodes = out.start || out.trace;
  // total stages = stage_off[n_plans] lives on the device; the caller sized
  // `work` with hapt_sim_workspace_bytes(total_stages, ring_depth), so the
  // ring region is what remains after the tail
  const size_t tail = sim_tail_bytes((size_t)n_plans);
  if (work_bytes < tail + 2 * (size_t)ring_depth * 8) {
    set_error("%s: workspace too small", who);
    return HAPT_ENOSPACE;
  }
  double *ring = (double *)work;
  char *wt = (char *)work + (work_bytes - tail);
  int32_t *perm = (int32_t *)wt;
  int32_t *cnt = (int32_t *)(wt + align_up((size_t)n_plans * 4));
  int32_t *bhist = cnt + 32;
  if (nodes && n_plans < 4096) {  // per-node outputs of a few plans: generic walk
    k_sim<<<grid_for(n_plans, 128), 128, 0, st>>>(n_plans, nullptr, nullptr, stage_off, t_fwd,
                                                  t_bwd, comm, counts, num_mb, makespan, out,
                                                  ring_depth, ring, status);
    ::hapt::note_launch();
    HAPT_LAUNCHED("k_sim");
    return HAPT_OK;
  }
  const int nb = (n_plans + kBucketBlock - 1) / kBucketBlock;
  k_bucket_hist<<<nb, kBucketBlock, 0, st>>>(n_plans, stage_off, bhist); ::hapt::note_launch();
  k_bucket_scan<<<1, 32, 0, st>>>(nb, bhist, cnt); ::hapt::note_launch();
  k_bucket_scatter<<<nb, kBucketBlock, 0, st>>>(n_plans, stage_off, bhist, cnt, perm); ::hapt::note_launch();
  int32_t h[19];  // [0..8] bucket sizes, [10..18] bucket starts in perm
  HAPT_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
  HAPT_CUDA(cudaStreamSynchronize(st));
  HAPT_LAUNCHED("k_bucket");
  // the eight per-S kernels are independent: run them concurrently on side
  // streams (each alone occupies the GPU only partially), joined back to st
  static thread_local cudaStream_t side[9];
  static thread_local cudaEvent_t ev[10];
  static thread_local bool init = false;
  if (!init) {
    for (int q = 1; q <= 8; ++q) {
      HAPT_CUDA(cudaStreamCreateWithFlags(&side[q], cudaStreamNonBlocking));
      HAPT_CUDA(cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming));
    }
    HAPT_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
    init = true;
  }
  HAPT_CUDA(cudaEventRecord(ev[0], st));
  // bucket 0 (S > 8) goes through the generic kernel below
#define HAPT_SIM_S(SV)                                                                        \
  if (h[SV] > 0) {                                                                            \
    HAPT_CUDA(cudaStreamWaitEvent(side[SV], ev[0], 0));                                       \
    launch_sim_s<SV>(perm + h[10 + SV], h[SV], stage_off, t_fwd, t_bwd, comm, counts, num_mb, \
                     makespan, status, out, side[SV]);                                         \
    HAPT_CUDA(cudaEventRecord(ev[SV], side[SV]));                                             \
    HAPT_CUDA(cudaStreamWaitEvent(st, ev[SV], 0));                                            \
  }
  HAPT_SIM_S(8) HAPT_SIM_S(7) HAPT_SIM_S(6) HAPT_SIM_S(5)
  HAPT_SIM_S(4) HAPT_SIM_S(3) HAPT_SIM_S(2) HAPT_SIM_S(1)
#undef HAPT_SIM_S
  HAPT_LAUNCHED("k_sim_s");
  // plans with S > 8 (bucket 0 = perm[0..h[0])) and any plan the fast path
  // handed back (appended after bucket 0) go through the generic walk
  HAPT_CUDA(cudaMemsetAsync(cnt + 20, 0, 4, st));
  if (h[0] > 0) {
    k_sim<<<grid_for(h[0], 128), 128, 0, st>>>(h[0], perm, cnt + 0, stage_off, t_fwd, t_bwd,
                                               comm, counts, num_mb, makespan, out, ring_depth,
                                               ring, status);
    ::hapt::note_launch();
  }
  k_sim_retry<<<grid_for(n_plans, 256), 256, 0, st>>>(n_plans, status, perm + h[0], cnt + 20); ::hapt::note_launch();
  k_sim<<<grid_for(n_plans, 128), 128, 0, st>>>(n_plans, perm + h[0], cnt + 20, stage_off,
                                                t_fwd, t_bwd, comm, counts, num_mb, makespan,
                                                out, ring_depth, ring, status);
  ::hapt::note_launch();
  HAPT_LAUNCHED("k_sim");
  return HAPT_OK;
}
}  // namespace

extern "C" int hapt_sim_1f1b(int32_t n_plans, const int32_t *stage_off, const double *t_fwd,
                             const double *t_bwd, const double *comm, const int32_t *counts,
                             const int32_t *num_mb, double *makespan, double *node_start,
                             double *node_end, const int64_t *node_off, int32_t ring_depth,
                             int32_t *status, void *work, size_t work_bytes, void *stream) {
  if (((node_start != nullptr) != (node_end != nullptr)) || (node_start && !node_off)) {
    set_error("hapt_sim_1f1b: invalid arguments");
    return HAPT_EINVAL;
  }
  return sim_1f1b("hapt_sim_1f1b", n_plans, stage_off, t_fwd, t_bwd, comm, counts, num_mb,
                  makespan, NodeOut{node_start, node_end, nullptr, node_off}, ring_depth, status,
                  work, work_bytes, stream);
}

extern "C" int hapt_sim_1f1b_trace(int32_t n_plans, const int32_t *stage_off,
                                   const double *t_fwd, const double *t_bwd, const double *comm,
                                   const int32_t *counts, const int32_t *num_mb,
                                   double *makespan, double *trace, const int64_t *trace_off,
                                   int32_t ring_depth, int32_t *status, void *work,
                                   size_t work_bytes, void *stream) {
  if (!trace || !trace_off || ((uintptr_t)trace & 15)) {
    set_error("hapt_sim_1f1b_trace: invalid arguments (trace must be 16-byte aligned)");
    return HAPT_EINVAL;
  }
  return sim_1f1b("hapt_sim_1f1b_trace", n_plans, stage_off, t_fwd, t_bwd, comm, counts,
                  num_mb, makespan,
                  NodeOut{nullptr, nullptr, reinterpret_cast<double2 *>(trace), trace_off},
                  ring_depth, status, work, work_bytes, stream);
}

extern "C" size_t hapt_dag_workspace_bytes(int32_t n_nodes) {
  return align_up((size_t)(n_nodes > 0 ? n_nodes : 1) * 4) * 3;
}

extern "C" int hapt_dag_longest_path(int32_t n_nodes, const int32_t *succ_off,
                                     const int32_t *succ_idx, const int32_t *indeg,
                                     const double *duration, double *start, double *end,
                                     double *makespan, int32_t *processed, void *work,
                                     size_t work_bytes, void *stream) {
  if (n_nodes < 1 || !succ_off || !succ_idx || !indeg || !duration || !start || !end ||
      !makespan || !processed || !work || work_bytes < hapt_dag_workspace_bytes(n_nodes)) {
    set_error("hapt_dag_longest_path: invalid arguments");
    return HAPT_EINVAL;
  }
  const size_t a = align_up((size_t)n_nodes * 4);
  char *w = (char *)work;
  k_dag<<<1, 1024, 0, (cudaStream_t)stream>>>(n_nodes, succ_off, succ_idx, indeg, duration,
                                               start, end, makespan, processed, (int32_t *)w,
                                               (int32_t *)(w + a), (int32_t *)(w + 2 * a)); ::hapt::note_launch();
  HAPT_LAUNCHED("k_dag");
  return HAPT_OK;
}

namespace {
int analyze_1f1b(const char *who, int32_t n_plans, int32_t total_stages,
                 const int32_t *stage_off, const double *t_fwd, const double *t_bwd,
                 const double *comm, const int32_t *counts, const int32_t *num_mb,
                 const double *mem_act, NodeIn in, const int32_t *status, double *stage_rep,
                 int32_t *peak_inflight, double *link_rep, double *steady_rate, void *stream) {
  if (n_plans < 1 || total_stages < 1 || !stage_off || !t_fwd || !t_bwd || !comm || !counts ||
      !num_mb || !in.off || !stage_rep || !peak_inflight || !link_rep || !steady_rate) {
    set_error("%s: invalid arguments", who);
    return HAPT_EINVAL;
  }
  const unsigned grid = grid_for(2 * (size_t)total_stages + n_plans, 128);
  if (in.trace)
    k_analyze<true><<<grid, 128, 0, (cudaStream_t)stream>>>(
        n_plans, stage_off, t_fwd, t_bwd, comm, counts, num_mb, mem_act, in, status, stage_rep,
        peak_inflight, link_rep, steady_rate);
  else
    k_analyze<false><<<grid, 128, 0, (cudaStream_t)stream>>>(
        n_plans, stage_off, t_fwd, t_bwd, comm, counts, num_mb, mem_act, in, status, stage_rep,
        peak_inflight, link_rep, steady_rate);
  ::hapt::note_launch();
  HAPT_LAUNCHED("k_analyze");
  return HAPT_OK;
}
}  // namespace

extern "C" int hapt_analyze_1f1b(int32_t n_plans, int32_t total_stages, const int32_t *stage_off,
                                 const double *t_fwd, const double *t_bwd, const double *comm,
                                 const int32_t *counts, const int32_t *num_mb,
                                 const double *mem_act, const double *node_start,
                                 const double *node_end, const int64_t *node_off,
                                 const int32_t *status, double *stage_rep,
                                 int32_t *peak_inflight, double *link_rep, double *steady_rate,
                                 void *stream) {
  if (!node_start || !node_end) {
    set_error("hapt_analyze_1f1b: invalid arguments");
    return HAPT_EINVAL;
  }
  return analyze_1f1b("hapt_analyze_1f1b", n_plans, total_stages, stage_off, t_fwd, t_bwd, comm,
                      counts, num_mb, mem_act, NodeIn{node_start, node_end, nullptr, node_off},
                      status, stage_rep, peak_inflight, link_rep, steady_rate, stream);
}

extern "C" int hapt_analyze_1f1b_trace(int32_t n_plans, int32_t total_stages,
                                       const int32_t *stage_off, const double *t_fwd,
                                       const double *t_bwd, const double *comm,
                                       const int32_t *counts, const int32_t *num_mb,
                                       const double *mem_act, const double *trace,
                                       const int64_t *trace_off, const int32_t *status,
                                       double *stage_rep, int32_t *peak_inflight,
                                       double *link_rep, double *steady_rate, void *stream) {
  if (!trace || ((uintptr_t)trace & 15)) {
    set_error("hapt_analyze_1f1b_trace: invalid arguments (trace must be 16-byte aligned)");
    return HAPT_EINVAL;
  }
  return analyze_1f1b("hapt_analyze_1f1b_trace", n_plans, total_stages, stage_off, t_fwd, t_bwd,
                      comm, counts, num_mb, mem_act,
                      NodeIn{nullptr, nullptr, reinterpret_cast<const double2 *>(trace),
                             trace_off},
                      status, stage_rep, peak_inflight, link_rep, steady_rate, stream);
}

extern "C" int hapt_steady_rate_1f1b(int32_t n_plans, const int32_t *stage_off,
                                     const int32_t *counts, const int32_t *num_mb,
                                     const double *node_start, const int64_t *node_off,
                                     const int32_t *rate_stage, const int32_t *status,
                                     double *steady_rate, void *stream) {
  if (n_plans < 1 || !stage_off || !counts || !num_mb || !node_start || !node_off ||
      !steady_rate) {
    set_error("hapt_steady_rate_1f1b: invalid arguments");
    return HAPT_EINVAL;
  }
  k_steady_rate<<<grid_for(n_plans, 128), 128, 0, (cudaStream_t)stream>>>(
      n_plans, stage_off, counts, num_mb, NodeIn{node_start, nullptr, nullptr, node_off},
      rate_stage, status, steady_rate);
  ::hapt::note_launch();
  HAPT_LAUNCHED("k_steady_rate");
  return HAPT_OK;
}

extern "C" size_t hapt_asap_workspace_bytes(int32_t n_nodes) {
  return n_nodes > 0 ? (size_t)n_nodes * 8 : 0;
}

extern "C" int hapt_dag_asap_check(int32_t n_nodes, const int32_t *succ_off,
                                   const int32_t *succ_idx, const int32_t *indeg,
                                   const double *duration, const double *start, double rel_tol,
                                   int32_t *first_bad, void *work, size_t work_bytes,
                                   void *stream) {
  if (n_nodes < 1 || !succ_off || !succ_idx || !indeg || !duration || !start || !first_bad ||
      !work || work_bytes < hapt_asap_workspace_bytes(n_nodes)) {
    set_error("hapt_dag_asap_check: invalid arguments");
    return HAPT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *hi = (unsigned long long *)work;
  HAPT_CUDA(cudaMemsetAsync(hi, 0, (size_t)n_nodes * 8, st));
  HAPT_CUDA(cudaMemcpyAsync(first_bad, &n_nodes, 4, cudaMemcpyHostToDevice, st));
  k_asap_max<<<grid_for(n_nodes, 256), 256, 0, st>>>(n_nodes, succ_off, succ_idx, duration,
                                                      start, hi);
  ::hapt::note_launch();
  k_asap_check<<<grid_for(n_nodes, 256), 256, 0, st>>>(n_nodes, indeg, start, hi, rel_tol,
                                                        first_bad);
  ::hapt::note_launch();
  HAPT_LAUNCHED("k_asap_check");
  return HAPT_OK;
}
