// K2 -- the stage-partition DP, batched over t_max candidates.
//
// Reference operator: meshpipe._core.dp_sweep (_dp.pyx:48-95), called once per
// candidate by planner.dp_search (planner.py:397-413).
//
//   F[s,k,g] = min over options o of mesh g_mesh[g] with opt_devs[o] <= g_avail[g],
//              and feasible spans i in CSR(o,k) (ascending), of
//              tt + (2c + F[s-1,i+1,g-devs])   subject to  tt <= t_max, c <= t_max,
//              F[s-1,..] finite, mp + kk*ma <= cap,  kk = ceil(2c/t_max)+1+N[s-1,i+1,g2]
//   ties: first strictly smaller in (o asc, i asc) order.
//
// B200 mapping:
//  * layer-synchronous sweep: F[s] reads only F[s-1], so one launch per layer
//    processes every (k,g) cell of every candidate in the batch;
//  * a warp = one cell for 32 candidates: lanes are candidates, so the loop
//    over (o, i) is warp-uniform, the CSR entry loads are broadcasts, and each
//    lane runs exactly the reference's scan order with strict '<' -- tie
//    semantics are preserved by construction, no cross-lane argmin needed;
//  * the previous layer is kept as a per-(state, split) "successor" table
//    H = 2c + F[s-1] (+inf when F is infinite or c > t_max) and
//    KK = ceil(2c/t_max) + 1 + N[s-1], candidate-innermost so that a warp's
//    32 lanes read 256 contiguous bytes; it is written by the epilogue of the
//    previous layer's launch (fused; no separate pass);
//  * the masks tt <= t_max and mp + kk*ma <= cap become integer compares
//    (pool rank, exact integer memory threshold); a row suffix-min of the
//    rank lets a warp stop a row once no lane can accept a later span;
//  * provably infinite cells/transitions (g < s, L-k+1 < s, i > L-s+1,
//    g2 < s-1) are never visited.
#include <stdlib.h>

#include <algorithm>

#include "hapt_common.cuh"

namespace hapt {
namespace {

#ifdef HAPT_COUNT_WORK
__device__ unsigned long long g_layer[4096 * 8];  // per layer: tasks, empty, chunks,
                                                  // staged, kept by bound, kept after probe,
                                                  // finite cells
__device__ unsigned long long g_work[8];  // executed / admissible / improving lane-transitions,
                                          // -, cell-tasks, empty cells, all-infinite cells, staged chunks
#endif
#ifndef HAPT_KWARPS
#define HAPT_KWARPS 4
#endif
constexpr int kWarps = HAPT_KWARPS;  // warps (cells) per block
// dp_relax_compact: one-warp blocks (32 resident per SM at 64 registers), so
// a finished warp's slot is refilled at once instead of idling until the
// slowest warp of its block is done (round 2: C 2.19 -> 2.04 ms, D2 74.5 ->
// 69.0 ms with the grid rule of run_sweep)
#ifndef HAPT_KWARPS_C
#define HAPT_KWARPS_C 1
#endif
#ifndef HAPT_RELAX_MINB_C
#define HAPT_RELAX_MINB_C (32 / HAPT_KWARPS_C)
#endif
constexpr int kWarpsC = HAPT_KWARPS_C;  // warps per dp_relax_compact block
constexpr int kParts = 32;  // copies of the per-candidate state counters
#ifndef HAPT_GRID_DIV
#define HAPT_GRID_DIV 2300  // cell-tasks (L x G x groups) per warp-per-SM of dp_relax_compact's cap
#endif
#ifndef HAPT_GRID_DIV4
#define HAPT_GRID_DIV4 1800  // the same at 4 candidates per lane (D1 pool 4.73 -> 4.68 ms; at
                             // CPL 2 the D1 2-GPU share measured 3.16 -> 3.26 ms with 1800)
#endif
#ifndef HAPT_WIN_MINLEN
#define HAPT_WIN_MINLEN 1  // window hull also bounded by each option's shortest span
#endif  // window cells of one (group, state) per relax warp
#ifndef HAPT_RELAX_MINB
#define HAPT_RELAX_MINB 8  // resident blocks/SM (64 registers at 4 warps per block)
#endif

// Candidates per lane.  A group of 32*CPL candidates shares one warp per DP
// cell: the staged CSR entry, the address arithmetic and one vector load of
// the successor values serve CPL candidates at once.
// Two per lane once the first layer alone has ~3.5 full GPU loads of warps
// (148 SMs x 32 resident warps); below that, one per lane keeps more warps
// in flight (measured: D1/C faster with 2, B faster with 1).  HAPT_CPL=1|2|4
// overrides for experiments.
int cpl_for(const hapt_tables *t, int n_cand) {
  if (const char *e = getenv("HAPT_CPL")) {
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) return v;
  }
  // two candidates per lane halve the warps a layer needs but lengthen each
  // warp's chain; measured (tools/time_batch.py, D1 and C) they pay off once
  // a batch has more than ~240 candidates (7.5 groups of 32) on tables large
  // enough to fill the GPU -- below that the extra warps of CPL = 1 hide more
  // latency (D1: 16 candidates 2.55 -> 1.82 ms, 224 candidates 4.13 -> 3.79 ms)
  // With the lane-bound pruning the transition loop is short and the
  // per-cell work (row metadata, staging, epilogue) dominates, so four
  // candidates per lane pay off on large batches despite a few spilled
  // registers (D1 1,786: 9.3 -> 7.2 ms; D2 7,019: 217 -> 144 ms; below
  // ~1,000 candidates, or with too few warps per layer, CPL = 2 stays ahead)
  const long cells = (long)t->L * t->G;
  const long warps4 = cells * ((n_cand + 127) / 128);
  // (v18, tools/gpu/cpl.py: C's 1,688 candidates on 102 x 64 cells run
  // faster at 2, D1's 1,786 on 82 x 256 cells at 4)
  // (round 2, tools/gpu/cpl_sizes.py on D1 / C / D2 slices: two per lane win
  // from ~40 candidates once a layer has a few thousand cell-warps, e.g. D1
  // 38: 1.08 -> 0.89 ms, 192: 1.82 -> 1.72 ms, C 38: 0.265 -> 0.231 ms, D2 128:
  // 5.06 -> 3.69 ms; four win on D2 from 890 candidates (15.6 -> 11.5 ms) but
  // not on D1 at 890 (3.22 vs 3.60 ms); config B's small tables stay at one)
  if (warps4 >= 150000) return 4;
  const long warps2 = cells * ((n_cand + 63) / 64);
  return (warps2 >= 4096 && n_cand > 32) ? 2 : 1;
}

#ifndef HAPT_U4
#define HAPT_U4 2
#endif
#ifndef HAPT_PROBE_MIN
#define HAPT_PROBE_MIN 6  // kept entries above which a chunk is probed (round 2: 2 -> 6, D1 -0.8 %, C -1 %)
#endif
#ifndef HAPT_U2
#define HAPT_U2 4  // 2, 4 or 8 (a 32-entry stage must be a multiple)
#endif
template <int CPL>
struct Unroll {
  static constexpr int value = CPL >= 4 ? HAPT_U4 : HAPT_U2;  // successor loads in flight per warp
};

struct Batch {
  // tables
  const hapt_span *spans;
  const int32_t *span_srank;
  const uint16_t *row_kmin, *row_pos;
  const int32_t *span_off, *opt_off, *opt_devs, *g_mesh, *g_avail, *g_crow;
  const double *cb;    // cb_same rows then cb_next rows, [2*n_meshes][L+1]
  const double *pool;
  const int64_t *counters;
  int L, G, s_max, n_cand, n_groups, rows, cpl, cw;
  size_t hg;           // (G+1)*(L+1) successor entries per candidate group
  // per batch
  const double *tmax;  // [n_cand]
  double *tmax_pad;    // [n_groups*cw]
  int32_t *tcnt;       // [n_groups*cw]  #pool values <= t_max
  uint4 *rowmeta;      // [n_groups][rows] {span_off of the row, cut | kmin << 16,
                       //  span_off - first split (INT_MIN if the row's splits are
                       //  not consecutive), 0}:
                       // cut = entries of the row before its suffix-min pool rank
                       // reaches the group's largest bound, kmin = row_kmin (one
                       // 8-byte load per option in the cell prologue)
  uint8_t *kc;         // [n_groups][2*n_meshes][L+1][cw] ceil(2c/t_max)+1 of every
                       // boundary row entry, 0xFF where c > t_max (_dp.pyx:76-82)
  int cb_rows;         // 2*n_meshes
  int2 *irange[3];     // [n_groups][G+1] (min, max) split i whose successor entry
                       // (state g) is finite for some candidate of the group;
                       // layer s reads [(s-1)%3], writes [s%3], resets [(s+1)%3]
  uint32_t *spanlen;   // [n_groups][2][n_opts] 0xffff - shortest, longest admissible
                       // span length of an option (before the group's cut)
  int2 *wopt;          // [n_groups][G+1][32] per state and option j < 32 of its mesh:
                       // {lo | hi << 16, g2*(L+1)}, the admissible split range of the
                       // current layer (dp_window) and the successor row
  uint32_t *clist;     // [n_groups][ccap] (g << 16 | k) of the cells inside the
                       // current layer's windows, group-local compact order
  size_t ccap;         // L*G >= cells of any layer
  int32_t *gtot[2];    // [n_groups] window cells per group at layers of each
                       // parity, reserved by dp_window's warps; dp_window(s)
                       // zeroes the other parity's (last read by dp_relax(s-1));
                       // dp_relax_compact turns them into the compact cell
                       // index space it walks (a prefix in shared memory)
  int2 *gopt;          // [G+1][32] per state g and option j < 32 of its mesh:
                       // {o, g - devs_o} ({-1, -1} past the mesh's options, g2 = -1
                       // where devs_o exceeds the state's available devices)
  int4 *gmeta;         // [G+1] per state g: first option of its mesh, option count,
                       // available devices, successor boundary row (g_crow)
  uint32_t *spart;     // [kParts][n_groups*cw] finite-cell counts of windowed
                       // layers, spread over kParts copies (dp_states_reduce)
  int n_opts;
  int probe;           // best-first probe per staged chunk (HAPT_PROBE=0: off)
  double *H[2];        // [n_groups][G+1][L+1][cw]
  uint16_t *K[2];
  double *Hmin[2];     // [n_groups][G+1][L+1]: lower bound of H over the group's lanes
  double *ftop;
  unsigned long long *states;
  hapt_dp_full full;
};

struct WsLayout {
  size_t tmax_pad, tcnt, rowmeta, kc, ir[3], spanlen, wopt, clist, gtot[2], gopt, gmeta, spart,
      H0,
      H1, K0, K1, Hm0, Hm1, total;
};

WsLayout ws_layout(const hapt_tables *t, int n_cand, int cpl) {
  WsLayout w{};
  const size_t cw = 32 * (size_t)cpl;
  const size_t ng = (n_cand + cw - 1) / cw, np = ng * cw;
  const size_t hg = (size_t)(t->G + 1) * (t->L + 1);
  const size_t rows = (size_t)t->n_opts * (t->L + 2);
  size_t cur = 0;
  w.tmax_pad = cur; cur += align_up(np * 8);
  w.tcnt = cur; cur += align_up(np * 4);
  w.rowmeta = cur; cur += align_up(ng * rows * 16);
  w.kc = cur; cur += align_up(ng * 2 * t->n_meshes * (t->L + 1) * cw);
  for (int j = 0; j < 3; ++j) {
    w.ir[j] = cur;
    cur += align_up(ng * (t->G + 1) * sizeof(int2));
  }
  w.spanlen = cur; cur += align_up(ng * 2 * t->n_opts * 4);
  w.wopt = cur; cur += align_up(ng * (t->G + 1) * 32 * 8);
  w.clist = cur; cur += align_up(ng * (size_t)t->L * t->G * 4);
  w.gtot[0] = cur; cur += align_up(ng * 4);
  w.gtot[1] = cur; cur += align_up(ng * 4);
  w.gopt = cur; cur += align_up((size_t)(t->G + 1) * 32 * sizeof(int2));
  w.gmeta = cur; cur += align_up((t->G + 1) * sizeof(int4));
  w.spart = cur; cur += align_up(kParts * np * 4);
  w.H0 = cur; cur += align_up(ng * hg * cw * 8);
  w.H1 = cur; cur += align_up(ng * hg * cw * 8);
  w.K0 = cur; cur += align_up(ng * hg * cw * 2);
  w.K1 = cur; cur += align_up(ng * hg * cw * 2);
  w.Hm0 = cur; cur += align_up(ng * hg * 8);
  w.Hm1 = cur; cur += align_up(ng * hg * 8);
  w.total = cur;
  return w;
}

WsLayout ws_layout(const hapt_tables *t, int n_cand) {
  return ws_layout(t, n_cand, cpl_for(t, n_cand));
}

// Large batches run as two independent halves (whole candidate groups, the
// low-t_max half and the high-t_max half) on two side streams, so one
// half's per-layer window passes and tails overlap the other's work.  Both
// halves keep the full batch's candidates per lane.  Measured (profiles/r2,
// tools/gpu/envs.sh HAPT_SPLIT=0): D2 78.2 -> 73.6 ms, D3 506 -> 472 ms;
// D1 (14 groups) and smaller batches are faster unsplit (5.15 vs 5.52 ms),
// alternating groups between the halves measured worse than contiguous
// halves (D2 74.6, D3 481, D1 5.29 ms), and 3-4 parts no better than two
// (round 2, same box: D3 452.8 vs 452.7 ms, D2 68.0 vs 67.9 ms).  Off when
// full outputs are requested.
struct Split {
  int parts, cpl;
  int n[2];
  size_t ws[2];  // aligned workspace bytes of each part
};

Split split_plan(const hapt_tables *t, int n_cand, bool full, int cpl = 0) {
  Split sp{};
  sp.cpl = cpl ? cpl : cpl_for(t, n_cand);
  const int cw = 32 * sp.cpl, ng = (n_cand + cw - 1) / cw;
  static const bool on = [] {
    const char *e = getenv("HAPT_SPLIT");
    return !(e && e[0] == '0');
  }();
  if (on && !full && sp.cpl == 4 && ng >= 24) {
    sp.parts = 2;
    sp.n[0] = (ng / 2) * cw;
    sp.n[1] = n_cand - sp.n[0];
  } else {
    sp.parts = 1;
    sp.n[0] = n_cand;
  }
  for (int j = 0; j < sp.parts; ++j) sp.ws[j] = align_up(ws_layout(t, sp.n[j], sp.cpl).total);
  return sp;
}

__device__ __forceinline__ int upper_bound(const double *a, int n, double v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Per group: candidate padding, pool ranks, the per-row suffix-rank cut, and
// the layer-0 successor table: F[0, L+1, 0] = 0 (_dp.pyx:41) is the only
// finite base state.
constexpr int kPrepY = 16;  // dp_prep blocks per group (rows and boundary entries split)
__global__ void dp_prep(Batch b) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_gmax;
  const int group = blockIdx.x, part = blockIdx.y;
  const int cw = b.cw;
  if (threadIdx.x == 0) s_gmax = 0;
  __syncthreads();
  // pool ranks of the group's candidates (every block needs the largest)
  if (threadIdx.x < cw) {
    const int cand = group * cw + threadIdx.x;
    const double tm = b.tmax[cand < b.n_cand ? cand : b.n_cand - 1];
    const int cnt = upper_bound(b.pool, (int)b.counters[1], tm);
    if (part == 0) {
      b.tmax_pad[cand] = tm;
      b.tcnt[cand] = cnt;
    }
    atomicMax(&s_gmax, cnt);
  }
  if (part == 0) {
    if (threadIdx.x == 0) {
      b.gtot[0][group] = 0;
      b.gtot[1][group] = 0;
    }
    // No fill of the successor tables: every read is confined to a state's
    // finite-successor range (irange), so layer 1 reads only the base entry
    // (g2 = 0, i = L) written below, and every later entry is written by the
    // layer before the one that reads it.
    // finite-successor ranges: layer 0 has only (g2 = 0, i = L); the buffers
    // layers 1 and 2 write start empty
    for (int g = threadIdx.x; g <= b.G; g += blockDim.x) {
      const int2 empty = make_int2(0x7fffffff, -1);
      b.irange[0][(size_t)group * (b.G + 1) + g] = g == 0 ? make_int2(b.L, b.L) : empty;
      b.irange[1][(size_t)group * (b.G + 1) + g] = empty;
      b.irange[2][(size_t)group * (b.G + 1) + g] = empty;
    }
    if (group == 0)
      for (int g = threadIdx.x; g <= b.G; g += blockDim.x) {
        const int r = b.g_mesh[g];
        b.gmeta[g] = make_int4(b.opt_off[r], b.opt_off[r + 1] - b.opt_off[r], b.g_avail[g],
                               b.g_crow[g]);
      }
    for (int x = threadIdx.x; x < kParts * cw; x += blockDim.x)
      b.spart[(size_t)(x / cw) * b.n_groups * cw + (size_t)group * cw + x % cw] = 0u;
  }
  if (group == 0) {  // per (state, option j < 32): the option and its successor state
    const int n = (b.G + 1) * 32;
    const int x0 = n * part / kPrepY, x1 = n * (part + 1) / kPrepY;
    for (int x = x0 + threadIdx.x; x < x1; x += blockDim.x) {
      const int g = x >> 5, j = x & 31;
      const int r = b.g_mesh[g], o0 = b.opt_off[r], no = b.opt_off[r + 1] - o0;
      int2 v = make_int2(-1, -1);
      if (j < no) {
        const int devs = b.opt_devs[o0 + j];
        v = make_int2(o0 + j, devs <= b.g_avail[g] ? g - devs : -1);
      }
      b.gopt[x] = v;
    }
  }
  __syncthreads();
  // suffix-min ranks are non-decreasing along a row: first entry no candidate
  // of this group can accept (prank >= srank >= max tcnt) ends the row's scan.
  // Shortest / longest admissible span (before the cut) of each option, for
  // dp_window: entries are in ascending span end, so the row's first entry
  // is its shortest and the last one before the cut its longest (both kept
  // as maxima: 0xffff - shortest, longest; zeroed by dp_ftop_init).
  const int gm = s_gmax;
  const int r0 = (int)((long)b.rows * part / kPrepY), r1 = (int)((long)b.rows * (part + 1) / kPrepY);
  for (int row = r0 + threadIdx.x; row < r1; row += blockDim.x) {
    const int beg = b.span_off[row], end = b.span_off[row + 1];
    int lo = beg, hi = end;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (b.span_srank[mid] < gm) lo = mid + 1; else hi = mid;
    }
    // a row's feasible splits form one run i0, i0+1, ... (OOM bounds a span
    // from above, the imbalance test from both sides), so entry p of the
    // row ends at i0 + p and its successor needs no span load (staging);
    // d0 = span_off - i0, INT_MIN where the run has gaps (overrides)
    int d0 = (int)0x80000000;
    if (end > beg) {
      const int i0 = (int)b.spans[beg].i;
      if ((int)b.spans[end - 1].i - i0 + 1 == end - beg) d0 = beg - i0;
    }
    b.rowmeta[(size_t)group * b.rows + row] =
        make_uint4((unsigned)beg, (unsigned)(lo - beg) | ((unsigned)b.row_kmin[row] << 16),
                   (unsigned)d0, 0u);
    if (lo > beg) {
      const int o = row / (b.L + 2), k = row - o * (b.L + 2);
      atomicMax(b.spanlen + ((size_t)group * 2 + 0) * b.n_opts + o,
                (unsigned)(0xffff - ((int)b.spans[beg].i - k + 1)));
      atomicMax(b.spanlen + ((size_t)group * 2 + 1) * b.n_opts + o,
                (unsigned)((int)b.spans[lo - 1].i - k + 1));
    }
  }
  // the launch-bound increment of every boundary entry for every candidate:
  // kk = (ceil(2c/t_max) + 1) + N (_dp.pyx:82, same association); c > t_max
  // skips the transition (_dp.pyx:76-78) -> 0xFF
  const size_t nkc = (size_t)b.cb_rows * (b.L + 1) * cw;
  uint8_t *kc = b.kc + (size_t)group * nkc;
  const size_t x0 = nkc * part / kPrepY, x1 = nkc * (part + 1) / kPrepY;
  for (size_t x = x0 + threadIdx.x; x < x1; x += blockDim.x) {
    const size_t e = x / cw;
    const double c = b.cb[e];
    const double tm = b.tmax[min(group * cw + (int)(x % cw), b.n_cand - 1)];
    kc[x] = c <= tm ? (uint8_t)((int)ceil(__ddiv_rn(__dmul_rn(2.0, c), tm)) + 1) : (uint8_t)0xFF;
  }
  if (part != 0) return;
  double *H = b.H[0] + (size_t)group * b.hg * cw;
  uint16_t *K = b.K[0] + (size_t)group * b.hg * cw;
  if (threadIdx.x < cw) {
    const double tm = b.tmax[min(group * cw + (int)threadIdx.x, b.n_cand - 1)];
    const int row = b.g_crow[0];
    const double c = b.cb[(size_t)row * (b.L + 1) + b.L];
    const size_t e = (size_t)b.L * cw + threadIdx.x;  // g2 = 0, i = L
    H[e] = kInf;
    K[e] = 0;
    if (c <= tm) {
      const double c2 = __dmul_rn(2.0, c);
      H[e] = __dadd_rn(c2, 0.0);
      K[e] = (uint16_t)((int)ceil(__ddiv_rn(c2, tm)) + 1);
    }
  }
  if (threadIdx.x == 0) {  // its lane minimum: finite iff some lane accepts c
    const double c = b.cb[(size_t)b.g_crow[0] * (b.L + 1) + b.L];
    bool any = false;
    for (int j = 0; j < cw; ++j) any |= c <= b.tmax[min(group * cw + j, b.n_cand - 1)];
    b.Hmin[0][(size_t)group * b.hg + b.L] = any ? __dadd_rn(__dmul_rn(2.0, c), 0.0) : kInf;
  }
}

// Per (group, state g) at layer s: the hull of k whose cell (k, g) can have an
// admissible transition -- through option o only splits i in the previous
// layer's finite range [lo, hi] of g2 = g - devs, i <= L-s+1, and spans no
// longer than the option's longest admissible one qualify, so
// k in [lo - maxlen_o + 1, min(hi, L-s+1)].  Cells outside the hull are
// provably infinite and are never read by layer s+1 (its read range comes
// from cells that were finite), so dp_relax skips them without writing.
// Per layer and group: the window [klo, khi] of every state g (cells outside
// are provably infinite: no option can reach a finite successor from them),
// the compact enumeration of the cells inside, and the reset of the irange
// buffer layer s+1 writes (last read by layer s-1).  One warp per state
// (lane = option), kWinWarps states per block and blockIdx.y = group, so the
// per-state dependent-load chains of a layer run on many SMs at once; each
// warp reserves its state's cells in the group's list with one atomic (the
// order of states in the list does not matter: cells are independent).
// dp_relax_compact prefix-sums the group totals itself.
constexpr int kWinWarps = 4;  // states per dp_window block (one warp each)
__global__ void __launch_bounds__(kWinWarps * 32) dp_window(Batch b, int s) {
  pdl_wait();
  pdl_trigger();
  const int group = blockIdx.y;
  const int L = b.L, G = b.G, imax = L - s + 1;
  const int lane = threadIdx.x & 31;
  const int g = blockIdx.x * kWinWarps + (threadIdx.x >> 5);
  // one warp per state g, lane j = option gm.x + j (+32, ... for larger
  // meshes): every option's loads are independent, the hull is a warp min/max
  int klo = 0x7fff, khi = 0;
  if (g <= G && g >= s) {
    // option / successor state of lane j come precomputed (gopt), so the
    // chain is gopt -> irange / spanlen -> the warp's hull
    const int2 go = __ldg(b.gopt + (size_t)g * 32 + lane);
    const int4 gm = b.gmeta[g];
    int2 *wo = b.wopt + ((size_t)group * (G + 1) + g) * 32;
    auto option = [&](const int o, const int g2, const bool store) {
      if (g2 < s - 1) {  // (also devs > available: g2 = -1)
        if (store) wo[lane] = make_int2(1, 0);
        return;
      }
      const int2 fr = b.irange[(s - 1) % 3][(size_t)group * (G + 1) + g2];
      if (store)
        wo[lane] = make_int2(fr.x <= min(imax, fr.y) ? fr.x | (min(imax, fr.y) << 16) : 1,
                             g2 * (L + 1));
      const int mn = 0xffff - (int)__ldg(b.spanlen + ((size_t)group * 2 + 0) * b.n_opts + o);
      const int mx = (int)__ldg(b.spanlen + ((size_t)group * 2 + 1) * b.n_opts + o);
      // option o reaches a finite successor from cell k only through spans
      // (k, i) with i in [fr.x, min(fr.y, L-s+1)] and admissible length
      // i-k+1 in [minlen_o, maxlen_o]
      const int hi = min(imax, fr.y);
      if (fr.x > hi || mx == 0) return;
      klo = min(klo, max(1, fr.x - mx + 1));
#if HAPT_WIN_MINLEN
      khi = max(khi, hi - mn + 1);
#else
      (void)mn;
      khi = max(khi, hi);
#endif
    };
    if (go.x >= 0) option(go.x, go.y, true);
    for (int j = lane + 32; j < gm.y; j += 32) {  // meshes with more than 32 shapes
      const int o = gm.x + j;
      const int devs = __ldg(b.opt_devs + o);
      option(o, devs <= gm.z ? g - devs : -1, false);
    }
  }
  klo = __reduce_min_sync(0xffffffffu, klo);
  khi = __reduce_max_sync(0xffffffffu, khi);
  const int n = khi >= klo ? khi - klo + 1 : 0;
  if (g <= G) {
    int base = 0;
    if (lane == 0 && n > 0) base = atomicAdd(b.gtot[s & 1] + group, n);
    base = __shfl_sync(0xffffffffu, base, 0);
    uint32_t *cl = b.clist + (size_t)group * b.ccap + base;
    for (int t = lane; t < n; t += 32) cl[t] = ((unsigned)g << 16) | (unsigned)(klo + t);
    if (lane == 0) {
      b.irange[(s + 1) % 3][(size_t)group * (G + 1) + g] = make_int2(0x7fffffff, -1);
    }
  }
  // the next windowed layer's totals (last read by dp_relax(s-1), which completed)
  if (blockIdx.x == 0 && threadIdx.x == 0) b.gtot[(s + 1) & 1][group] = 0;
}

template <int CPL>
__device__ __forceinline__ void load_h(const char *p, double (&h)[CPL]) {
  if constexpr (CPL == 1) {
    h[0] = __ldg(reinterpret_cast<const double *>(p));
  } else {
#pragma unroll
    for (int c = 0; c < CPL; c += 2) {
      const double2 v = __ldg(reinterpret_cast<const double2 *>(p) + c / 2);
      h[c] = v.x;
      h[c + 1] = v.y;
    }
  }
}

template <int CPL>
__device__ __forceinline__ void load_k(const char *p, int (&k)[CPL]) {
  if constexpr (CPL == 1) {
    k[0] = __ldg(reinterpret_cast<const uint16_t *>(p));
  } else if constexpr (CPL == 2) {
    const unsigned v = __ldg(reinterpret_cast<const unsigned *>(p));
    k[0] = v & 0xffff;
    k[1] = v >> 16;
  } else {
    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
    k[0] = v.x & 0xffff;
    k[1] = v.x >> 16;
    k[2] = v.y & 0xffff;
    k[3] = v.y >> 16;
  }
}

// The transitions of one cell, flattened over its admissible (option, split)
// entries in the reference's order (o ascending, i ascending, _dp.pyx:58,67)
// and staged in shared memory as
//     {tt (2 words), w2 = prank*2048 + o, w3 = byte offset of the successor}
// so `tt <= t_max` is `w2 < cnt*2048` (o < 2048) and the option of the
// winner rides along for free.  The stage is padded to a multiple of the
// unroll with inert entries (w2 = ~0 never passes), so the loop has no
// guards.  Every candidate keeps the first strict minimum, exactly the
// reference's `cand < best` update.
__device__ __forceinline__ void prefetch_l1(const void *p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <bool WITH_KK, int CPL>
__device__ __forceinline__ void relax_entries(const int4 *__restrict__ st,
                                              const uint16_t *__restrict__ skm, int n,
                                              const unsigned (&cnt)[CPL],
                                              const char *__restrict__ Hb,
                                              const char *__restrict__ Kb, double (&bv)[CPL],
                                              unsigned (&bw3)[CPL]) {
  constexpr int U = Unroll<CPL>::value;
  // At 4 candidates per lane ptxas issues a step's second entry's loads only
  // after the first entry's adds (register limit), so each entry waits a
  // full L2 round trip; the next step's rows are prefetched to L1 instead
  // (no registers held) and its loads then hit L1 (D1 pool 5.04 -> 4.82 ms;
  // at CPL 2 the step's loads are already in flight together and a prefetch
  // only costs: C 2.08 -> 2.22 ms).
  constexpr int PF = CPL == 4 ? U : 0;
  for (int u = 0; u < n; u += U) {
    int4 ex[U];
    double h[U][CPL];
    int kk[U][CPL];
#pragma unroll
    for (int q = 0; q < (PF ? U : 0); ++q)
      if (u + PF + q < n) {
        const unsigned w = (unsigned)st[u + PF + q].w;
        prefetch_l1(Hb + w);
        if (WITH_KK) prefetch_l1(Kb + (w >> 2));
      }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      ex[q] = st[u + q];
      load_h<CPL>(Hb + (unsigned)ex[q].w, h[q]);
      if (WITH_KK) load_k<CPL>(Kb + ((unsigned)ex[q].w >> 2), kk[q]);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const double tt = __hiloint2double(ex[q].y, ex[q].x);
      const int km = WITH_KK ? (int)skm[u + q] : 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double v = __dadd_rn(tt, h[q][c]);  // tt + (2c + F)  (_dp.pyx:85)
#ifdef HAPT_COUNT_WORK  // instrumented build only (tools/work_counts.py)
        if (u + q < n) {
          const bool adm = (unsigned)ex[q].z < cnt[c] && h[q][c] != kInf;
          atomicAdd(&g_work[0], 1ull);
          if (adm) atomicAdd(&g_work[1], 1ull);
          if (adm && v < bv[c]) atomicAdd(&g_work[2], 1ull);
        }
#endif
        if ((unsigned)ex[q].z < cnt[c] && (!WITH_KK || kk[q][c] <= km) && v < bv[c]) {
          bv[c] = v;
          bw3[c] = (unsigned)ex[q].w;
        }
      }
    }
  }
}

// Per-lane option data of state g at layer s that does not depend on the
// cell's k: lane j holds option o0 + c0 + j of mesh g_mesh[g].  Computed once
// per chunk of cells of one (group, g) and reused by every cell of the chunk
// (the opt_devs -> irange part of the per-cell dependent-load chain).
struct OptLane {
  int fr;     // lo | hi << 16: split range of the successor state g2 = g - devs
              // whose entries are finite for some candidate (empty: lo > hi)
  int hbase;  // g2 * (L+1): successor row of g2
};

__device__ __forceinline__ OptLane opt_lane(const Batch &b, int s, int group, int g, int o,
                                            int avail, bool valid) {
  OptLane ol;
  ol.fr = 1;
  ol.hbase = 0;
  if (valid) {
    const int devs = __ldg(b.opt_devs + o), g2 = g - devs;
    if (devs <= avail && g2 >= s - 1) {
      // admissible splits: inside the range where state g2's successor entry
      // is finite for some candidate of the group (the rest are ones the
      // reference skips for all these candidates: fc == inf)
      const int2 fr = b.irange[(s - 1) % 3][(size_t)group * (b.G + 1) + g2];
      const int hi = min(b.L - s + 1, fr.y);
      ol.fr = fr.x <= hi ? fr.x | (hi << 16) : 1;
      ol.hbase = g2 * (b.L + 1);
    }
  }
  return ol;
}

// Option of a cell's winner, for backpointers only (the transition loop
// tracks just the winner's successor).  The winner is the first entry in the
// reference's order (o ascending, then i) with the minimum value; every entry
// through the winning successor (g2 = g - devs, split i) shares its H, so the
// winner's option is the first option of the mesh with devs devices whose
// span (k, i) is admissible for this candidate (tt <= t_max, KK <= kmax) and
// whose value tt + H equals the best (_dp.pyx:58-91, strict '<' update).
__device__ __noinline__ int winner_option(const int32_t *opt_devs, const int32_t *span_off,
                                          const hapt_span *spans, int L, int k, int devs, int i,
                                          double best, unsigned cnt, int kk, double h, int o0,
                                          int nopt) {
  for (int o = o0; o < o0 + nopt; ++o) {
    if (opt_devs[o] != devs) continue;
    const int row = o * (L + 2) + k;
    int lo = span_off[row], hi = span_off[row + 1];
    while (lo < hi) {  // entries ascend in span end i
      const int mid = (lo + hi) >> 1;
      if ((int)spans[mid].i < i) lo = mid + 1; else hi = mid;
    }
    if (lo == span_off[row + 1] || (int)spans[lo].i != i) continue;
    const hapt_span e = spans[lo];
    if ((unsigned)e.prank < cnt && kk <= (int)e.kmax && __dadd_rn(e.tt, h) == best) return o;
  }
  return -1;  // unreachable for a recorded winner
}

// One DP cell (k, g) of layer s for the 32*CPL candidates of `group`, executed
// by one warp: fin[c] = whether the cell is finite for candidate c; writes the
// successor entry of layer s+1 and, for a finite entry, widens irange.
// ol0: opt_lane() of the mesh's first 32 options (lane j = option o0 + j).
template <int CPL>
__device__ __forceinline__ void relax_cell(const Batch &b, int s, int group, int k, int g,
                                           int lane, int4 *__restrict__ stage_e,
                                           uint16_t *__restrict__ stage_k, int (&fin)[CPL],
                                           const int o0, const int nopt, const OptLane &ol0) {
  constexpr int CW = 32 * CPL;
  const int L = b.L, G = b.G;
  const int cand0 = group * CW + lane * CPL;
  unsigned cnt[CPL];  // #pool values <= t_max: tt <= t_max <=> prank < cnt
#pragma unroll
  for (int c = 0; c < CPL; ++c) cnt[c] = (unsigned)b.tcnt[cand0 + c];
  const size_t gbase = (size_t)group * b.hg;
  const double *Hg = b.H[(s - 1) & 1] + gbase * CW + lane * CPL;
  const uint16_t *Kg = b.K[(s - 1) & 1] + gbase * CW + lane * CPL;
  const char *Hb = reinterpret_cast<const char *>(Hg);
  const char *Kb = reinterpret_cast<const char *>(Kg);
  double bv[CPL];
  unsigned bw3[CPL];  // successor byte offset of the winner (its option: winner_option)
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    bv[c] = kInf;
    bw3[c] = 0;
  }
  // options of mesh r, 32 at a time (a mesh rarely has more than 32 submesh
  // shapes); rows are visited in ascending option order
  // (one chunk in practice: the second and later only for meshes with more
  // than 32 shapes, so nothing of the chunk loop stays live in the main path)
  auto chunk = [&](const int c0, const OptLane &ol) {
    const int nch = min(32, nopt - c0);
    const int o = o0 + c0 + lane;
    // lane j: admissible entries of option o's row (k) at this layer
    int len = 0, beg = 0, d0 = (int)0x80000000;
    bool needkk = false;
    const int lo_i = max(k, ol.fr & 0xffff), hi_i = (int)((unsigned)ol.fr >> 16);
    if (lane < nch && lo_i <= hi_i) {
      const int row = o * (L + 2) + k;
      // admissible splits also end at i <= L-s+1 (later successors are
      // provably infinite) and before the group's suffix-rank cut
      const uint4 rm = __ldg(b.rowmeta + (size_t)group * b.rows + row);
      const int soff = (int)rm.x, cut = (int)(rm.y & 0xffffu), kmin = (int)(rm.y >> 16);
      d0 = (int)rm.z;
      const uint16_t *pos = b.row_pos + (size_t)row * (L + 2);
      const int a = __ldg(pos + lo_i - 1);
      const int z = min((int)__ldg(pos + hi_i), cut);
      beg = soff + a;
      len = max(0, z - a);
      // KK <= 3s at layer s: ceil(2c/t_max) <= 2 and N grows by <= 3 per
      // stage, so a row whose thresholds are all >= 3s cannot fail the
      // memory mask (_dp.pyx:83)
      needkk = len > 0 && kmin < 3 * s;
    }
    const int hbase = ol.hbase;
    int incl = len;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    const int T = __shfl_sync(0xffffffffu, incl, 31);
    const int start = incl - len;
    // successor of flattened entry t of this row = hsp + t (consecutive
    // splits), so its bound load need not wait for the span entry
    const int hsp = d0 != (int)0x80000000 ? hbase + beg - start - d0 : (int)0x80000000;
#ifdef HAPT_COUNT_WORK
    if (lane == 0 && c0 == 0) {
      atomicAdd(&g_work[4], 1ull);
      if (T == 0 && nopt <= 32) atomicAdd(&g_work[5], 1ull);
      atomicAdd(&g_work[7], (unsigned long long)((T + 31) / 32));
      atomicAdd(&g_layer[s * 8 + 0], 1ull);
      if (T == 0) atomicAdd(&g_layer[s * 8 + 1], 1ull);
      atomicAdd(&g_layer[s * 8 + 2], (unsigned long long)((T + 31) / 32));
      atomicAdd(&g_layer[s * 8 + 3], (unsigned long long)T);
    }
#endif
    const bool anykk = __any_sync(0xffffffffu, needkk);
    const double *Hm = b.Hmin[(s - 1) & 1] + gbase;
    for (int r0 = 0; r0 < T; r0 += 32) {
      const int t = r0 + lane;
      // A transition's value tt + H[lane] (H = 2c + F >= 0) is at least
      // tt + Hmin (a lower bound of H over the group's lanes), and an update needs a strict
      // improvement; an entry with tt + Hmin >= every lane's current best
      // cannot change any lane's winner and is not staged (bv only falls,
      // so the bound taken here holds for the whole chunk).
      // max over lanes via the high words (non-negative doubles order like
      // their bit patterns): hi:ffffffff bounds every best from above
      unsigned mh = 0;
#pragma unroll
      for (int c = 0; c < CPL; ++c) mh = max(mh, (unsigned)__double2hiint(bv[c]));
      mh = __reduce_max_sync(0xffffffffu, mh);
      const double bmax = mh >= 0x7ff00000u ? kInf : __hiloint2double((int)mh, -1);
      // owner row: number of rows whose entries end at or before t, by binary
      // search over the lanes' inclusive ends (non-decreasing; rows past nch
      // end at T > t for every real entry)
      int j = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, j + step - 1);
        if (v <= t) j += step;
      }
      const int jj = min(j, 31);
      const int ob = __shfl_sync(0xffffffffu, beg, jj);
      const int os = __shfl_sync(0xffffffffu, start, jj);
      const int oh = __shfl_sync(0xffffffffu, hbase, jj);
      const int hs = __shfl_sync(0xffffffffu, hsp, jj);
      int4 se = make_int4(0, 0, -1, 0);  // inert padding entry
      uint16_t sk = 0;
      bool keep = false;
      double lb = kInf;  // tt + Hmin: no lane's value through this entry is lower
      if (t < T) {
        double hmv = 0.0;
        // (at CPL 4 the early bound load measured slower: 4.76 -> 5.05 ms on D1)
        const bool spec = CPL < 4 && hs != (int)0x80000000;
        if (spec) hmv = __ldg(Hm + hs + t);
        const int4 x = __ldg(reinterpret_cast<const int4 *>(b.spans + ob + (t - os)));
        const int succ = oh + (x.w & 0xffff);
        if (!spec) hmv = __ldg(Hm + succ);
        lb = __dadd_rn(__hiloint2double(x.y, x.x), hmv);
        keep = lb < bmax;
        // w2 = pool rank (INT32_MAX for a non-finite t: never below a count)
        se = make_int4(x.x, x.y, x.z, succ * (256 * CPL));
        sk = (uint16_t)((unsigned)x.w >> 16);
      }
      // Best-first probe: evaluate the kept entry with the smallest bound
      // (position f) for every lane without recording it, which tightens the
      // bound to bn = max over lanes of min(best, probe).  Every lane's final
      // best is <= bn, so an entry after f with lb >= bn, or before f with
      // lb > bn, is never the first minimum and is dropped; f itself stays
      // and is relaxed in its own place, so the scan order is the reference's.
      unsigned kept = __ballot_sync(0xffffffffu, keep);
#ifdef HAPT_COUNT_WORK
      if (lane == 0) atomicAdd(&g_layer[s * 8 + 4], (unsigned long long)__popc(kept));
#endif
      if (b.probe && __popc(kept) > HAPT_PROBE_MIN) {
        const unsigned lh = keep ? (unsigned)__double2hiint(lb) : 0xffffffffu;
        const unsigned ml = __reduce_min_sync(0xffffffffu, lh);
        const int f = __ffs(__ballot_sync(0xffffffffu, keep && lh == ml)) - 1;
        const int px = __shfl_sync(0xffffffffu, se.x, f), py = __shfl_sync(0xffffffffu, se.y, f);
        const unsigned pz = __shfl_sync(0xffffffffu, (unsigned)se.z, f);
        const unsigned pw = __shfl_sync(0xffffffffu, (unsigned)se.w, f);
        const int pk = __shfl_sync(0xffffffffu, (int)sk, f);
        double hp[CPL];
        int kp[CPL];
        load_h<CPL>(Hb + pw, hp);
        if (anykk) load_k<CPL>(Kb + (pw >> 2), kp);
        const double pt = __hiloint2double(py, px);
        unsigned mh = 0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          double m = bv[c];
          const double v = __dadd_rn(pt, hp[c]);  // never NaN: tt, H >= 0 (or +inf)
          if (pz < cnt[c] && (!anykk || kp[c] <= pk) && v < m) m = v;
          mh = max(mh, (unsigned)__double2hiint(m));
        }
        mh = __reduce_max_sync(0xffffffffu, mh);
        const double bn = mh >= 0x7ff00000u ? kInf : __hiloint2double((int)mh, -1);
        keep = keep && (lane == f || (lane < f ? lb <= bn : lb < bn));
        kept = __ballot_sync(0xffffffffu, keep);
      }
      // kept entries first, in order, padded with inert entries to a multiple
      // of the transition loop's unroll
      const unsigned below = kept & ((1u << lane) - 1u);
      const int n = __popc(kept);
#ifdef HAPT_COUNT_WORK
      if (lane == 0) atomicAdd(&g_layer[s * 8 + 5], (unsigned long long)n);
#endif
      constexpr int U = Unroll<CPL>::value;
      if (keep) {
        stage_e[__popc(below)] = se;
        stage_k[__popc(below)] = sk;
      } else if (n + (lane - __popc(below)) < (n + U - 1) / U * U) {
        stage_e[n + (lane - __popc(below))] = make_int4(0, 0, -1, 0);
        stage_k[n + (lane - __popc(below))] = 0;
      }
      __syncwarp();
      if (anykk)
        relax_entries<true, CPL>(stage_e, stage_k, n, cnt, Hb, Kb, bv, bw3);
      else
        relax_entries<false, CPL>(stage_e, stage_k, n, cnt, Hb, Kb, bv, bw3);
      __syncwarp();
    }
  };
  chunk(0, ol0);
  if (nopt > 32) {
    const int avail = b.gmeta[g].z;
    for (int c0 = 32; c0 < nopt; c0 += 32)
      chunk(c0, opt_lane(b, s, group, g, o0 + c0 + lane, avail, lane < min(32, nopt - c0)));
  }
  // A warp with no finite best records nothing, and its successor entry is
  // infinite for every lane: only Hmin = +inf is written, which makes the
  // next layer drop every transition into it at staging (lb = +inf is never
  // below a bound), so its H / K slots are never read and need no write.
  // (ftop / N / bp keep their initial +inf / 0 / -1.)  A third of D1's cells
  // end this way.
  const size_t hm_idx = gbase + (size_t)g * (L + 1) + (k - 1);
  {
    bool any = false;
#pragma unroll
    for (int c = 0; c < CPL; ++c) any |= bv[c] < kInf;
    if (!__any_sync(0xffffffffu, any)) {
#pragma unroll
      for (int c = 0; c < CPL; ++c) fin[c] = 0;
      if (lane == 0) b.Hmin[s & 1][hm_idx] = kInf;
#ifdef HAPT_COUNT_WORK
      if (lane == 0) atomicAdd(&g_work[6], 1ull);
#endif
      return;
    }
  }
  // epilogue per candidate
  double hn[CPL];
  int kn[CPL], bkk[CPL];
  const int crow = __ldg(&b.gmeta[g].w);  // successor boundary row of state g
  const double c2 = crow >= 0 ? __dmul_rn(2.0, b.cb[(size_t)crow * (L + 1) + (k - 1)]) : 0.0;
  const uint8_t *kcp = b.kc + ((size_t)group * b.cb_rows + (crow >= 0 ? crow : 0)) * (L + 1) * CW +
                       (size_t)(k - 1) * CW + lane * CPL;
  // the CPL launch-bound increments of this lane in one load (0xFF: c > t_max)
  unsigned kcw = 0xFFFFFFFFu;
  if (crow >= 0) {
    if constexpr (CPL == 4) kcw = __ldg(reinterpret_cast<const unsigned *>(kcp));
    else if constexpr (CPL == 2) kcw = 0xFFFF0000u | __ldg(reinterpret_cast<const uint16_t *>(kcp));
    else kcw = 0xFFFFFF00u | __ldg(kcp);
  }
  // N of the winner = its KK (_dp.pyx:87); reloaded once instead of tracked
  // (the successor's K slot is at byte offset bw3 / 4 from Kb)
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    fin[c] = bv[c] < kInf;
    bkk[c] = fin[c] ? (int)__ldg(reinterpret_cast<const uint16_t *>(Kb + (bw3[c] >> 2)) + c) : 0;
  }
  if (k == 1 && g == G) {  // warp-uniform: the top cell F[s,1,G] of every candidate
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int cand = cand0 + c;
      if (cand >= b.n_cand) continue;
      b.ftop[(size_t)cand * (b.s_max + 1) + s] = bv[c];
      if (b.full.ntop) b.full.ntop[(size_t)cand * (b.s_max + 1) + s] = bkk[c];
    }
  }
  // warp-uniform: backpointers / F / N are only recorded when a caller asked
  if (b.full.bp_packed != nullptr || b.full.bp_o != nullptr) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int cand = cand0 + c;
      if (!fin[c] || cand >= b.n_cand) continue;
      const int boff = (int)(bw3[c] / (256u * CPL));
      const int g2 = boff / (L + 1), bi = boff - g2 * (L + 1);
      const int bo = winner_option(b.opt_devs, b.span_off, b.spans, L, k, g - g2, bi, bv[c],
                                   cnt[c], bkk[c], __ldg(Hg + (size_t)boff * CW + c), o0, nopt);
      const size_t e = (((size_t)cand * (b.s_max + 1) + s) * (L + 2) + k) * (G + 1) + g;
      if (b.full.bp_packed) b.full.bp_packed[e] = (bo << 16) | bi;
      if (b.full.bp_o) {
        if (b.full.F) b.full.F[e] = bv[c];
        if (b.full.N) b.full.N[e] = (double)bkk[c];
        b.full.bp_i[e] = bi;
        b.full.bp_o[e] = bo;
      }
    }
  }
  // successor entry (state g, split i = k-1) for layer s+1:
  // H = 2c + F, KK = (ceil(2c/t_max) + 1) + N, or +inf if c > t_max
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const int kcv = (int)((kcw >> (8 * c)) & 0xFFu);
    const bool ok = fin[c] && kcv != 0xFF;
    hn[c] = ok ? __dadd_rn(c2, bv[c]) : kInf;
    kn[c] = ok ? kcv + bkk[c] : 0;
  }
  const size_t o_idx = hm_idx * CW + lane * CPL;
  bool anyfin = false;
  unsigned hh = 0xffffffffu;  // min over lanes of the high words; hi:0 bounds every H below
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    anyfin |= hn[c] != kInf;
    hh = min(hh, (unsigned)__double2hiint(hn[c]));
  }
  hh = __reduce_min_sync(0xffffffffu, hh);
  if (lane == 0) b.Hmin[s & 1][hm_idx] = __hiloint2double((int)hh, 0);
  const bool wfin = __any_sync(0xffffffffu, anyfin);
#ifdef HAPT_COUNT_WORK
  if (lane == 0 && wfin) atomicAdd(&g_layer[s * 8 + 6], 1ull);
#endif
  if (wfin) {  // otherwise Hmin = +inf already shields the slots (see above)
    double *ho = b.H[s & 1] + o_idx;
    uint16_t *ko = b.K[s & 1] + o_idx;
    if constexpr (CPL == 1) {
      ho[0] = hn[0];
      ko[0] = (uint16_t)kn[0];
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 2)
        reinterpret_cast<double2 *>(ho)[c / 2] = make_double2(hn[c], hn[c + 1]);
      if constexpr (CPL == 2)
        *reinterpret_cast<unsigned *>(ko) = (unsigned)kn[0] | ((unsigned)kn[1] << 16);
      else
        *reinterpret_cast<uint2 *>(ko) = make_uint2((unsigned)kn[0] | ((unsigned)kn[1] << 16),
                                                    (unsigned)kn[2] | ((unsigned)kn[3] << 16));
    }
  }
  if (wfin && lane == 0) {
    int2 *fr = &b.irange[s % 3][(size_t)group * (G + 1) + g];
    atomicMin(&fr->x, k - 1);
    atomicMax(&fr->y, k - 1);
  }
}

template <int CPL>
__global__ void __launch_bounds__(kWarps * 32, HAPT_RELAX_MINB)
    dp_relax(Batch b, int s, int group0, unsigned long long nk_magic) {
  pdl_wait();
  pdl_trigger();
  constexpr int CW = 32 * CPL;
  __shared__ int fin_cnt[kWarps][CW];
  __shared__ int4 stage_e[kWarps][32];
  __shared__ uint16_t stage_k[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int group = group0 + blockIdx.y;
  const int L = b.L, G = b.G;
  const int nk = L - s + 1, ng = G - s + 1;
  const int cell = blockIdx.x * kWarps + warp;
  // cell / nk by multiply-high with ceil(2^32/nk): exact for cell < 2^20,
  // nk < 2^12 (hapt_tables_init bounds both)
  const int gq = (int)(((unsigned long long)(unsigned)cell * nk_magic) >> 32);
  const int k = 1 + cell - gq * nk;
  const int g = s + gq;
  const bool active = cell < nk * ng;
  int fin[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) fin[c] = 0;
  if (active) {
    const int4 gm = b.gmeta[g];
    const OptLane ol0 = opt_lane(b, s, group, g, gm.x + lane, gm.z, lane < gm.y);
    relax_cell<CPL>(b, s, group, k, g, lane, stage_e[warp], stage_k[warp], fin, gm.x, gm.y,
                    ol0);
  }
  if (blockIdx.x == 0) {  // the buffer layer s+1 writes: last read by layer s-1
    for (int x = threadIdx.x; x <= G; x += blockDim.x)
      b.irange[(s + 1) % 3][(size_t)group * (G + 1) + x] = make_int2(0x7fffffff, -1);
  }
#pragma unroll
  for (int c = 0; c < CPL; ++c) fin_cnt[warp][lane * CPL + c] = fin[c];
  __syncthreads();
  for (int x = threadIdx.x; x < CW; x += blockDim.x) {
    int sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sum += fin_cnt[w][x];
    const int cand = group * CW + x;
    if (sum && cand < b.n_cand) atomicAdd(&b.states[cand], (unsigned long long)sum);
  }
}

// Warp-collective cursor over the compact cell index space of a layer: the
// groups' window cells (gtot, dp_window) concatenated in group order.  A
// warp's cells come in increasing index order, so the cursor only moves
// forward, 32 groups at a time: lane j holds the inclusive prefix of group
// base + j within the chunk (run = cells of the groups before the chunk).
struct GroupCursor {
  int base, run, incl, tot;
  __device__ __forceinline__ void load(const int32_t *gtot, int ng, int lane) {
    const int j = base + lane;
    const int v = j < ng ? __ldg(gtot + j) : 0;
    incl = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    tot = __shfl_sync(0xffffffffu, incl, 31);
  }
  // group owning cell idx (< the layer's total) and the index of the
  // group's first cell
  __device__ __forceinline__ int find(const int32_t *gtot, int ng, int idx, int lane,
                                      int &first) {
    if (idx < run) {  // (a claim that wrapped around to an earlier segment)
      base = 0;
      run = 0;
      load(gtot, ng, lane);
    }
    while (idx >= run + tot) {
      run += tot;
      base += 32;
      load(gtot, ng, lane);
    }
    const int j = __popc(__ballot_sync(0xffffffffu, run + incl <= idx));
    const int ex = __shfl_sync(0xffffffffu, incl, (j + 31) & 31);
    first = run + (j == 0 ? 0 : ex);
    return base + j;
  }
};

// Windowed layers: only the cells inside dp_window's windows, enumerated
// compactly, one warp per cell over a grid of one-warp blocks (capped per SM
// by run_sweep) that strides over the list -- no warp is spent on a provably
// infinite cell, and
// the state's per-option split ranges come precomputed from dp_window.
// Finite-cell counts stay in shared memory while a warp's cells stay in one
// group and go to one of kParts counter copies (dp_states_reduce sums them)
// when it changes, so no warp waits at a block barrier for a slower one.
template <int CPL>
__global__ void __launch_bounds__(kWarpsC * 32, HAPT_RELAX_MINB_C)
    dp_relax_compact(Batch b, int s) {
  pdl_wait();
  pdl_trigger();
  constexpr int CW = 32 * CPL;
  __shared__ int4 stage_e[kWarpsC][32];
  __shared__ uint16_t stage_k[kWarpsC][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t *gtot = b.gtot[s & 1];
  const int ng = b.n_groups;
  GroupCursor gc{0, 0, 0, 0};
  gc.load(gtot, ng, lane);
  // the layer's total: the sum over every chunk of 32 groups
  int total = gc.tot;
  for (int j0 = 32; j0 < ng; j0 += 32) {
    const int v = j0 + lane < ng ? __ldg(gtot + j0 + lane) : 0;
    total += __reduce_add_sync(0xffffffffu, v);
  }
  uint32_t *part = b.spart + (size_t)(blockIdx.x & (kParts - 1)) * b.n_groups * CW;
  // this warp's finite-cell counts of its current group (shared memory, not
  // registers: the cell body is at the 64-register limit)
  __shared__ unsigned s_cnt[kWarpsC][CW];
  unsigned *cnt = &s_cnt[warp][lane * CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) cnt[c] = 0u;
  int cur = -1;
  auto flush = [&](int grp) {
    uint32_t *dst = part + (size_t)grp * CW + lane * CPL;
    if constexpr (CPL == 1) {
      if (cnt[0]) atomicAdd(dst, cnt[0]);
    } else {
#pragma unroll
      for (int c = 0; c < CPL; c += 2)
        if (cnt[c] | cnt[c + 1])
          atomicAdd(reinterpret_cast<unsigned long long *>(dst + c),
                    (unsigned long long)cnt[c] | ((unsigned long long)cnt[c + 1] << 32));
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) cnt[c] = 0u;
  };
  auto cell = [&](const int idx) {
    int first;
    const int group = gc.find(gtot, ng, idx, lane, first);
    if (group != cur) {
      if (cur >= 0) flush(cur);
      cur = group;
    }
    const unsigned gk = __ldg(b.clist + (size_t)group * b.ccap + (idx - first));
    const int g = (int)(gk >> 16), k = (int)(gk & 0xffffu);
    const int4 gm = b.gmeta[g];
    // this layer's split ranges of the state's first 32 options (dp_window)
    OptLane ol0;
    {
      const int2 w = lane < gm.y ? __ldg(b.wopt + ((size_t)group * (b.G + 1) + g) * 32 + lane)
                                 : make_int2(1, 0);
      ol0.fr = w.x;
      ol0.hbase = w.y;
    }
    int fin[CPL];
    relax_cell<CPL>(b, s, group, k, g, lane, stage_e[warp], stage_k[warp], fin, gm.x, gm.y, ol0);
#pragma unroll
    for (int c = 0; c < CPL; ++c) cnt[c] += fin[c] ? 1u : 0u;
  };
  for (int idx = blockIdx.x * kWarpsC + warp; idx < total; idx += gridDim.x * kWarpsC) cell(idx);
  if (cur >= 0) flush(cur);
}

// states[cand] += sum of the kParts partial counters (padding lanes dropped)
__global__ void dp_states_reduce(Batch b) {
  pdl_wait();
  pdl_trigger();
  const int np = b.n_groups * b.cw;
  for (int cand = blockIdx.x * blockDim.x + threadIdx.x; cand < b.n_cand;
       cand += gridDim.x * blockDim.x) {
    unsigned long long sum = 0;
#pragma unroll 8
    for (int q = 0; q < kParts; ++q) sum += b.spart[(size_t)q * np + cand];
    if (sum) b.states[cand] += sum;
  }
}

__global__ void dp_ftop_init(double *ftop, unsigned long long *states, int n_cand, int s_max,
                             uint32_t *spanlen, int n_span) {
  pdl_wait();
  pdl_trigger();
  const long x = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x < (long)n_cand * (s_max + 1)) ftop[x] = kInf;
  if (x < n_cand) states[x] = 0;
  if (x < n_span) spanlen[x] = 0u;
}

// Per candidate best s and T* (planner.py:287-298), then the lexicographic
// (T*, index) argmin == ParallelPlan.sort_key order over the pool.
__global__ void dp_select(const double *ftop, const double *tmax, int n_cand, int s_max,
                          long long B, double *tstar, int32_t *best_s, int32_t *winner) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  double bv = kInf;
  int bidx = -1;
  const double bm1 = (double)(B - 1);
  for (int c = threadIdx.x; c < n_cand; c += blockDim.x) {
    const double tm = tmax[c];
    const double pen = __dmul_rn(bm1, tm);
    double best_total = kInf;
    int bs = -1;
    for (int s = 1; s <= s_max; ++s) {
      const double v = ftop[(size_t)c * (s_max + 1) + s];
      if (!isfinite(v)) continue;
      const double total = __dadd_rn(v, pen);
      if (total < best_total) {
        best_total = total;
        bs = s;
      }
    }
    tstar[c] = best_total;
    best_s[c] = bs;
    if (bs >= 0 && (bidx < 0 || best_total < bv)) {  // c ascends: ties keep first
      bv = best_total;
      bidx = c;
    }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bidx;
  __syncthreads();
  for (int w = blockDim.x / 2; w; w >>= 1) {
    if (threadIdx.x < w) {
      const int j = threadIdx.x + w;
      const bool take = si[j] >= 0 && (si[threadIdx.x] < 0 || sv[j] < sv[threadIdx.x] ||
                                       (sv[j] == sv[threadIdx.x] && si[j] < si[threadIdx.x]));
      if (take) {
        sv[threadIdx.x] = sv[j];
        si[threadIdx.x] = si[j];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) winner[0] = si[0];
}

// Backpointer walk (planner.py:300-312) + the K chain (planner.py:330-338).
__global__ void dp_walk(hapt_dp_full full, const int32_t *opt_devs, int L, int G, int s_max,
                        int best_s, int32_t *stages, int32_t *kchain, int32_t *n_stages,
                        int32_t *err) {
  if (threadIdx.x || blockIdx.x) return;
  int s = best_s, k = 1, g = G, n = 0;
  *err = 0;
  while (s > 0) {
    const size_t e = ((size_t)s * (L + 2) + k) * (G + 1) + g;
    const int i = full.bp_i[e], o = full.bp_o[e];
    if (i < 0) {
      *err = 1;
      break;
    }
    stages[3 * n + 0] = k;
    stages[3 * n + 1] = i;
    stages[3 * n + 2] = o;
    kchain[n] = (int)full.N[e];
    ++n;
    g -= opt_devs[o];
    k = i + 1;
    --s;
  }
  if (!*err && (k != L + 1 || g != 0)) *err = 2;
  *n_stages = n;
}

// Backpointer walk over packed (o << 16 | i) backpointers (planner.py:300-312).
__global__ void dp_walk_packed(const int32_t *bp, const int32_t *opt_devs, int L, int G,
                               int best_s, int32_t *stages, int32_t *n_stages) {
  if (threadIdx.x || blockIdx.x) return;
  int s = best_s, k = 1, g = G, n = 0;
  while (s > 0) {
    const int v = bp[((size_t)s * (L + 2) + k) * (G + 1) + g];
    const int o = v >> 16, i = v & 0xffff;
    if (i < k || i > L || o < 0) {
      *n_stages = -1;
      return;
    }
    stages[3 * n + 0] = k;
    stages[3 * n + 1] = i;
    stages[3 * n + 2] = o;
    ++n;
    g -= opt_devs[o];
    k = i + 1;
    --s;
  }
  *n_stages = (k != L + 1 || g != 0) ? -2 : n;
}

__global__ void fill_full(hapt_dp_full f, size_t n, int L, int G) {
  const size_t x = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  if (f.F) f.F[x] = (x == (size_t)(L + 1) * (G + 1)) ? 0.0 : kInf;
  if (f.N) f.N[x] = 0.0;
  f.bp_i[x] = -1;
  f.bp_o[x] = -1;
}

__global__ void k_rank_hist(const hapt_span *spans, const int64_t *counters,
                            unsigned long long *hist) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= counters[0]) return;
  const int pr = spans[idx].prank;
  if (pr != 0x7fffffff) atomicAdd(&hist[pr], 1ull);
}

__global__ void k_activated(const double *pool, const int64_t *counters,
                            unsigned long long *hist, const double *tmax, int n_cand,
                            int64_t *out) {
  // single block: in-place exclusive scan of hist[0..plen], then
  // activated(t) = #entries with rank < upper_bound(pool, t) = hist[cnt]
  __shared__ unsigned long long part[1024];
  const int plen = (int)counters[1];
  const int n = plen + 1;
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  unsigned long long sum = 0;
  for (int i = lo; i < hi; ++i) sum += hist[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const unsigned long long v = part[i];
      part[i] = run;
      run += v;
    }
  }
  __syncthreads();
  unsigned long long run = part[threadIdx.x];
  for (int i = lo; i < hi; ++i) {
    const unsigned long long v = hist[i];
    hist[i] = run;
    run += v;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < n_cand; c += blockDim.x)
    out[c] = (int64_t)hist[upper_bound(pool, plen, tmax[c])];
}

Batch make_batch(const hapt_tables *t, const double *tmax, int n_cand, double *ftop,
                 int64_t *states, const hapt_dp_full *full, void *work, int cpl = 0) {
  if (cpl == 0) cpl = cpl_for(t, n_cand);
  WsLayout w = ws_layout(t, n_cand, cpl);
  char *wb = (char *)work;
  Batch b{};
  b.spans = t->spans;
  b.span_srank = t->span_srank;
  b.row_kmin = t->row_kmin;
  b.row_pos = t->row_pos;
  b.rows = t->n_opts * (t->L + 2);
  b.span_off = t->span_off;
  b.opt_off = t->opt_off;
  b.opt_devs = t->opt_devs;
  b.g_mesh = t->g_mesh;
  b.g_avail = t->g_avail;
  b.g_crow = t->g_crow;
  b.cb = t->cb_same;
  b.pool = t->pool;
  b.counters = t->counters;
  b.L = t->L;
  b.G = t->G;
  b.s_max = t->s_max;
  b.n_cand = n_cand;
  b.cpl = cpl;
  {
    static const int probe = getenv("HAPT_PROBE") ? atoi(getenv("HAPT_PROBE")) : 1;
    b.probe = probe;
  }
  b.cw = 32 * b.cpl;
  b.n_groups = (n_cand + b.cw - 1) / b.cw;
  b.hg = (size_t)(t->G + 1) * (t->L + 1);
  b.tmax = tmax;
  b.tmax_pad = (double *)(wb + w.tmax_pad);
  b.tcnt = (int32_t *)(wb + w.tcnt);
  b.rowmeta = (uint4 *)(wb + w.rowmeta);
  b.kc = (uint8_t *)(wb + w.kc);
  b.cb_rows = 2 * t->n_meshes;
  for (int j = 0; j < 3; ++j) b.irange[j] = (int2 *)(wb + w.ir[j]);
  b.spanlen = (uint32_t *)(wb + w.spanlen);
  b.wopt = (int2 *)(wb + w.wopt);
  b.clist = (uint32_t *)(wb + w.clist);
  b.ccap = (size_t)t->L * t->G;
  b.gtot[0] = (int32_t *)(wb + w.gtot[0]);
  b.gtot[1] = (int32_t *)(wb + w.gtot[1]);
  b.gopt = (int2 *)(wb + w.gopt);
  b.spart = (uint32_t *)(wb + w.spart);
  b.gmeta = (int4 *)(wb + w.gmeta);
  b.n_opts = t->n_opts;
  b.H[0] = (double *)(wb + w.H0);
  b.H[1] = (double *)(wb + w.H1);
  b.K[0] = (uint16_t *)(wb + w.K0);
  b.K[1] = (uint16_t *)(wb + w.K1);
  b.Hmin[0] = (double *)(wb + w.Hm0);
  b.Hmin[1] = (double *)(wb + w.Hm1);
  b.ftop = ftop;
  b.states = (unsigned long long *)states;
  if (full) b.full = *full;
  return b;
}

// The sweep is a chain of ~2 launches per layer; every kernel of it is
// enqueued with programmatic dependent launch (waits for its predecessor on
// the device, so the launch gap overlaps the previous kernel's tail).
int run_sweep(const Batch &b, cudaStream_t st) {
  // measured: on tiny tables (config A, L*G ~ 100) the dependent-launch wait
  // costs more than the gap it hides; kernel timing (prof_on) brackets every
  // launch with events, so it runs without PDL
  const bool pdl = pdl_enabled() && (long)b.L * b.G >= 4096 && !prof_on();
  const int n_span = 2 * b.n_groups * b.n_opts;
  {
    ProfScope ps(kProfOther, st);
    HAPT_CUDA(launch_pdl(dp_ftop_init,
                         grid_for(max((size_t)b.n_cand * (b.s_max + 1), (size_t)n_span), 256),
                         256, st, pdl, b.ftop, b.states, b.n_cand, b.s_max, b.spanlen, n_span));
  }
  {
    ProfScope ps(kProfOther, st);  // block >= 128 = max group width
    HAPT_CUDA(launch_pdl(dp_prep, dim3(b.n_groups, kPrepY), 256, st, pdl, b));
  }
  // SM count of this device (dp_relax_compact's grid cap, per layer below)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  unsigned gcap = 0;  // per layer below, unless HAPT_RELAX_GRID fixes it
  if (const char *e = getenv("HAPT_RELAX_GRID")) {
    const long v = atol(e);
    if (v >= 1 && v <= (1l << 20)) gcap = (unsigned)v;
  }
  static const long win_min = [] {
    const char *e = getenv("HAPT_WINDOW_MIN");
    const long v = e ? atol(e) : 32768;
    return v >= 0 ? v : 32768;
  }();
  for (int s = 1; s <= b.s_max; ++s) {
    const long cells = (long)(b.L - s + 1) * (b.G - s + 1);
    if (cells <= 0) break;
    const unsigned gx = grid_for(cells, kWarps);
    const unsigned long long nk = (unsigned long long)(b.L - s + 1);
    const unsigned long long magic = ((1ull << 32) + nk - 1) / nk;  // ceil(2^32 / nk)
    // the window pass pays off once the layer has far more warps than the
    // GPU holds at once; on small grids its launch costs more than it saves
    const int use_window = cells * b.n_groups >= win_min;
    if (use_window) {
      const dim3 wgrid((b.G + 1 + kWinWarps - 1) / kWinWarps, b.n_groups);
      {
        ProfScope ps(kProfWindow, st);
        HAPT_CUDA(launch_pdl(dp_window, wgrid, kWinWarps * 32, st, pdl, b, s));
      }
      // The list's length is only known on the device: the grid is capped at
      // a number of warps per SM that grows with the batch (L x G x groups /
      // 2,300, between 64 and 192 per SM), and the warps stride over the
      // list.  Surplus warps exit at once but still cost their dispatch; too
      // few leave the tail unbalanced.  Measured with one-warp blocks
      // (tools/gpu/grid_sweep.sh): D1 pool (294 K) 128 / SM 5.03 ms vs 256 / SM
      // 5.20; D2 (1.1 M per half) 192 / SM 68.3 ms; D1 8-GPU share (73 K)
      // 64 / SM 1.30 ms vs 128 / SM 1.47 ms.
      unsigned cap = gcap;
      if (cap == 0) {
        const long wps =
            (std::min(192l, std::max(64l, (long)b.L * b.G * b.n_groups /
                                              (b.cpl == 4 ? HAPT_GRID_DIV4 : HAPT_GRID_DIV))) +
             16) / 32 * 32;
        cap = (unsigned)(wps / kWarpsC) * (unsigned)sms;
      }
      const unsigned cgrid = min(cap, grid_for((size_t)cells * b.n_groups, kWarpsC));
      const dim3 blk(kWarpsC * 32);
      ProfScope ps(kProfRelax, st);
      if (b.cpl == 1)
        HAPT_CUDA(launch_pdl(dp_relax_compact<1>, cgrid, blk, st, pdl, b, s));
      else if (b.cpl == 2)
        HAPT_CUDA(launch_pdl(dp_relax_compact<2>, cgrid, blk, st, pdl, b, s));
      else
        HAPT_CUDA(launch_pdl(dp_relax_compact<4>, cgrid, blk, st, pdl, b, s));
      continue;
    }
    for (int g0 = 0; g0 < b.n_groups; g0 += 65535) {
      const dim3 grid(gx, min(65535, b.n_groups - g0)), blk(kWarps * 32);
      ProfScope ps(kProfRelax, st);
      if (b.cpl == 1)
        HAPT_CUDA(launch_pdl(dp_relax<1>, grid, blk, st, pdl, b, s, g0, magic));
      else if (b.cpl == 2)
        HAPT_CUDA(launch_pdl(dp_relax<2>, grid, blk, st, pdl, b, s, g0, magic));
      else
        HAPT_CUDA(launch_pdl(dp_relax<4>, grid, blk, st, pdl, b, s, g0, magic));
    }
  }
  ProfScope ps(kProfOther, st);
  HAPT_CUDA(launch_pdl(dp_states_reduce, grid_for(b.n_cand, 256), 256, st, pdl, b));
  return HAPT_OK;
}

}  // namespace
}  // namespace hapt

using namespace hapt;

extern "C" size_t hapt_dp_workspace_bytes(const hapt_tables *t, int32_t n_cand) {
  if (!t || n_cand < 1) return 0;
  // enough for any candidates-per-lane choice (hapt_dp_sweep_batch_cpl)
  size_t best = 0;
  for (const int cpl : {1, 2, 4}) {
    const Split sp = split_plan(t, n_cand, false, cpl);
    size_t total = 0;
    for (int j = 0; j < sp.parts; ++j) total += sp.ws[j];
    best = max(best, max(total, align_up(ws_layout(t, n_cand, cpl).total)));  // (full: one part)
  }
  return best;
}

namespace {
// side streams of the calling host thread on the current device (fork/join
// of a split sweep; the caller's stream orders everything around them)
struct SideStreams {
  int dev = -1;
  cudaStream_t s[2] = {nullptr, nullptr};
};
thread_local SideStreams t_side;

int side_streams(cudaStream_t (&out)[2]) {
  int dev = 0;
  HAPT_CUDA(cudaGetDevice(&dev));
  if (t_side.dev != dev) {
    for (int j = 0; j < 2; ++j)
      HAPT_CUDA(cudaStreamCreateWithFlags(&t_side.s[j], cudaStreamNonBlocking));
    t_side.dev = dev;  // (streams of a previous device stay alive: rare)
  }
  out[0] = t_side.s[0];
  out[1] = t_side.s[1];
  return HAPT_OK;
}
}  // namespace

extern "C" int hapt_dp_sweep_batch(const hapt_tables *t, const double *tmax, int32_t n_cand,
                                   double *ftop, int64_t *states, const hapt_dp_full *full,
                                   void *work, size_t work_bytes, void *stream) {
  return hapt_dp_sweep_batch_cpl(t, tmax, n_cand, ftop, states, full, work, work_bytes, 0, stream);
}

extern "C" int hapt_dp_sweep_batch_cpl(const hapt_tables *t, const double *tmax, int32_t n_cand,
                                       double *ftop, int64_t *states, const hapt_dp_full *full,
                                       void *work, size_t work_bytes, int32_t cpl, void *stream) {
  if (!t || !tmax || n_cand < 1 || !ftop || !states || !work ||
      !(cpl == 0 || cpl == 1 || cpl == 2 || cpl == 4)) {
    set_error("hapt_dp_sweep_batch: invalid arguments");
    return HAPT_EINVAL;
  }
  if (full && ((full->bp_o == nullptr) != (full->bp_i == nullptr) ||
               ((full->F || full->N) && !full->bp_o))) {
    set_error("hapt_dp_sweep_batch: F/N need bp_i and bp_o, which go together");
    return HAPT_EINVAL;
  }
  if (cpl == 0 || getenv("HAPT_CPL")) cpl = cpl_for(t, n_cand);  // (HAPT_CPL: experiments)
  const Split sp = split_plan(t, n_cand, full != nullptr, cpl);
  size_t need = 0;
  for (int j = 0; j < sp.parts; ++j) need += sp.ws[j];
  if (work_bytes < need) {
    set_error("hapt_dp_sweep_batch: workspace %zu < %zu", work_bytes, need);
    return HAPT_ENOSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (sp.parts == 1) {
    Batch b = make_batch(t, tmax, n_cand, ftop, states, full, work, sp.cpl);
    return run_sweep(b, st);
  }
  cudaStream_t side[2];
  if (const int rc = side_streams(side)) return rc;
  cudaEvent_t fork, done[2];
  HAPT_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  HAPT_CUDA(cudaEventRecord(fork, st));
  char *w = (char *)work;
  int off = 0;
  for (int j = 0; j < 2; ++j) {
    HAPT_CUDA(cudaStreamWaitEvent(side[j], fork, 0));
    Batch b = make_batch(t, tmax + off, sp.n[j], ftop + (size_t)off * (t->s_max + 1),
                         states + off, nullptr, w, sp.cpl);
    const int rc = run_sweep(b, side[j]);
    if (rc != HAPT_OK) return rc;
    HAPT_CUDA(cudaEventCreateWithFlags(&done[j], cudaEventDisableTiming));
    HAPT_CUDA(cudaEventRecord(done[j], side[j]));
    HAPT_CUDA(cudaStreamWaitEvent(st, done[j], 0));
    w += sp.ws[j];
    off += sp.n[j];
  }
  // events are released once the work they mark has completed
  cudaEventDestroy(fork);
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  return HAPT_OK;
}

extern "C" int hapt_dp_select(const double *ftop, const double *tmax, int32_t n_cand,
                              int32_t s_max, int64_t num_microbatches, double *tstar,
                              int32_t *best_s, int32_t *winner, void *stream) {
  if (!ftop || !tmax || n_cand < 1 || !tstar || !best_s || !winner) {
    set_error("hapt_dp_select: invalid arguments");
    return HAPT_EINVAL;
  }
  dp_select<<<1, 1024, 0, (cudaStream_t)stream>>>(ftop, tmax, n_cand, s_max,
                                                   (long long)num_microbatches, tstar,
                                                   best_s, winner); ::hapt::note_launch();
  HAPT_LAUNCHED("dp_select");
  return HAPT_OK;
}

namespace {
struct BtLayout {
  size_t tmax, ftop, states, err, bpi, bpo, N, ws, total;
};
BtLayout bt_layout(const hapt_tables *t) {
  BtLayout y{};
  const size_t cells = (size_t)(t->s_max + 1) * (t->L + 2) * (t->G + 1);
  size_t cur = 0;
  y.tmax = cur; cur += align_up(8);
  y.ftop = cur; cur += align_up((size_t)(t->s_max + 1) * 8);
  y.states = cur; cur += align_up(8);
  y.err = cur; cur += align_up(4);
  y.bpi = cur; cur += align_up(cells * 4);
  y.bpo = cur; cur += align_up(cells * 4);
  y.N = cur; cur += align_up(cells * 8);
  y.ws = cur; cur += align_up(ws_layout(t, 1).total);
  y.total = cur;
  return y;
}
}  // namespace

extern "C" size_t hapt_backtrack_workspace_bytes(const hapt_tables *t) {
  if (!t) return 0;
  return bt_layout(t).total;
}

extern "C" int hapt_dp_backtrack(const hapt_tables *t, double tmax, int32_t best_s,
                                 int32_t *stages, int32_t *kchain, int32_t *n_stages,
                                 void *work, size_t work_bytes, void *stream) {
  if (!t || !stages || !kchain || !n_stages || !work || best_s < 1 || best_s > t->s_max) {
    set_error("hapt_dp_backtrack: invalid arguments");
    return HAPT_EINVAL;
  }
  BtLayout y = bt_layout(t);
  if (work_bytes < y.total) {
    set_error("hapt_dp_backtrack: workspace %zu < %zu", work_bytes, y.total);
    return HAPT_ENOSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char *w = (char *)work;
  double *d_tmax = (double *)(w + y.tmax);
  HAPT_CUDA(cudaMemcpyAsync(d_tmax, &tmax, 8, cudaMemcpyHostToDevice, st));
  hapt_dp_full full{};
  full.F = nullptr;
  full.N = (double *)(w + y.N);
  full.bp_i = (int32_t *)(w + y.bpi);
  full.bp_o = (int32_t *)(w + y.bpo);
  const size_t cells = (size_t)(t->s_max + 1) * (t->L + 2) * (t->G + 1);
  fill_full<<<grid_for(cells, 256), 256, 0, st>>>(full, cells, t->L, t->G); ::hapt::note_launch();
  Batch b = make_batch(t, d_tmax, 1, (double *)(w + y.ftop), (int64_t *)(w + y.states), &full,
                       w + y.ws);
  int rc = run_sweep(b, st);
  if (rc != HAPT_OK) return rc;
  int32_t *err = (int32_t *)(w + y.err);
  dp_walk<<<1, 32, 0, st>>>(full, t->opt_devs, t->L, t->G, t->s_max, best_s, stages, kchain,
                            n_stages, err); ::hapt::note_launch();
  HAPT_LAUNCHED("dp_walk");
  int32_t herr = 0;
  HAPT_CUDA(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
  HAPT_CUDA(cudaStreamSynchronize(st));
  if (herr) {
    set_error(herr == 1 ? "broken backpointer chain"
                        : "plan does not cover all layers and devices");
    return HAPT_ECHAIN;
  }
  return HAPT_OK;
}

namespace {
struct OneLayout {
  size_t tmax, ftop, states, ws, total;
};
OneLayout one_layout(const hapt_tables *t) {
  OneLayout y{};
  size_t cur = 0;
  y.tmax = cur; cur += align_up(8);
  y.ftop = cur; cur += align_up((size_t)(t->s_max + 1) * 8);
  y.states = cur; cur += align_up(8);
  y.ws = cur; cur += align_up(ws_layout(t, 1).total);
  y.total = cur;
  return y;
}
}  // namespace

extern "C" size_t hapt_dp_sweep_workspace_bytes(const hapt_tables *t) {
  return t ? one_layout(t).total : 0;
}

extern "C" int hapt_dp_sweep(const hapt_tables *t, double tmax, double *F, double *N,
                             int32_t *bp_i, int32_t *bp_o, void *work, size_t work_bytes,
                             void *stream) {
  if (!t || !F || !N || !bp_i || !bp_o || !work || !(tmax > 0.0)) {
    set_error("hapt_dp_sweep: invalid arguments");
    return HAPT_EINVAL;
  }
  const OneLayout y = one_layout(t);
  if (work_bytes < y.total) {
    set_error("hapt_dp_sweep: workspace %zu < %zu", work_bytes, y.total);
    return HAPT_ENOSPACE;
  }
  cudaStream_t st = (cudaStream_t)stream;
  char *w = (char *)work;
  double *d_tmax = (double *)(w + y.tmax);
  HAPT_CUDA(cudaMemcpyAsync(d_tmax, &tmax, 8, cudaMemcpyHostToDevice, st));
  // the reference's fresh output arrays: F = +inf but F[0, L+1, 0] = 0,
  // N = 0, bp = -1 (_dp.pyx:33-41); the sweep writes every finite cell
  hapt_dp_full full{};
  full.F = F, full.N = N, full.bp_i = bp_i, full.bp_o = bp_o;
  const size_t cells = (size_t)(t->s_max + 1) * (t->L + 2) * (t->G + 1);
  fill_full<<<grid_for(cells, 256), 256, 0, st>>>(full, cells, t->L, t->G);
  ::hapt::note_launch();
  HAPT_LAUNCHED("fill_full");
  Batch b = make_batch(t, d_tmax, 1, (double *)(w + y.ftop), (int64_t *)(w + y.states), &full,
                       w + y.ws);
  return run_sweep(b, st);
}

extern "C" int hapt_dp_walk(const hapt_tables *t, const int32_t *bp_cand, int32_t best_s,
                            int32_t *stages, int32_t *n_stages, void *stream) {
  if (!t || !bp_cand || !stages || !n_stages || best_s < 1 || best_s > t->s_max) {
    set_error("hapt_dp_walk: invalid arguments");
    return HAPT_EINVAL;
  }
  dp_walk_packed<<<1, 32, 0, (cudaStream_t)stream>>>(bp_cand, t->opt_devs, t->L, t->G, best_s,
                                                     stages, n_stages); ::hapt::note_launch();
  HAPT_LAUNCHED("dp_walk_packed");
  return HAPT_OK;
}

extern "C" int hapt_activated_pairs(const hapt_tables *t, const double *tmax, int32_t n_cand,
                                    int64_t *activated, void *stream) {
  if (!t || !tmax || n_cand < 1 || !activated) {
    set_error("hapt_activated_pairs: invalid arguments");
    return HAPT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // the rank histogram lives in the tables scratch
  unsigned long long *hist = (unsigned long long *)tables_hist(t);
  HAPT_CUDA(cudaMemsetAsync(hist, 0, ((size_t)t->pool_cap + 1) * 8, st));
  k_rank_hist<<<grid_for(t->nnz_cap, 256), 256, 0, st>>>(t->spans, t->counters, hist); ::hapt::note_launch();
  k_activated<<<1, 1024, 0, st>>>(t->pool, t->counters, hist, tmax, n_cand, activated); ::hapt::note_launch();
  HAPT_LAUNCHED("hapt_activated_pairs");
  return HAPT_OK;
}

#ifdef HAPT_COUNT_WORK
extern "C" int hapt_debug_layers(unsigned long long *out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, hapt::g_layer, sizeof(unsigned long long) * 4096 * 8) ==
                 cudaSuccess
             ? HAPT_OK
             : HAPT_ECUDA;
}
// instrumented build only: cumulative transition counters of the DP loop
extern "C" int hapt_debug_work(unsigned long long *out) {
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, hapt::g_work, sizeof(unsigned long long) * 8) == cudaSuccess
             ? HAPT_OK
             : HAPT_ECUDA;
}
#endif
