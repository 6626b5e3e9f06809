// K1 -- cost tables on the device.
//
// Replaces, bit for bit:
//   ProfileStore._build + analytic_profile   (profiling.py:88-103, 212-286)
//   boundary_costs                           (profiling.py:128-147)
//   DpTables.__init__                        (planner.py:169-248)
//   feasible_t_values / candidate_tmax       (profiling.py:315-318; planner.py:424-429)
//
// Design: every (option, q, p) cell is one thread.  The reference's
// structural dedup ("one profile per distinct (signature, mesh, shape) key,
// first span in q-major order is canonical", profiling.py:241-251) becomes a
// canonical-start table canon_q[q][p] computed from longest-common-prefix
// runs of the layer-signature ids; an alias cell then evaluates exactly the
// expressions its canonical cell evaluates (same inputs, same rounding), so
// no cross-thread dependency exists.  The CSR feasible-span index, its
// per-entry DP metadata (integer memory threshold, pool rank, row suffix-min
// rank) and the sorted-unique t_max pool are produced by hapt_tables_finalize,
// which the drop-in dp_sweep path shares.
#include <cub/cub.cuh>

#include "hapt_common.cuh"

namespace hapt {
namespace {

constexpr unsigned long long kPadKey = ~0ull;
constexpr size_t kCubTempBase = 64ull << 20;

struct Layout {
  size_t cells, rows, nnz_cap, pool_cap;
  size_t off[40];
  size_t total;
};

// Order-preserving map of doubles onto unsigned keys (radix-sort transform).
__device__ __forceinline__ unsigned long long fkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double fdecode(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

Layout layout(int L, int G, int n_opts, int n_meshes) {
  Layout y{};
  y.cells = (size_t)n_opts * (L + 2) * (L + 2);
  y.rows = (size_t)n_opts * (L + 2);
  y.nnz_cap = (size_t)n_opts * L * (L + 1) / 2;
  if (y.nnz_cap < 1) y.nnz_cap = 1;
  y.pool_cap = y.nnz_cap;
  size_t sz[40];
  int n = 0;
  for (int i = 0; i < 7; ++i) sz[n++] = y.cells * 8;      // 0..6 dense tables
  sz[n++] = y.cells;                                      // 7 cell_state
  sz[n++] = (size_t)(L + 2) * (L + 2) * 4;                // 8 canon_q
  sz[n++] = (size_t)n_opts * 8;                           // 9 opt_cap
  sz[n++] = (size_t)n_opts * 4;                           // 10 opt_mesh
  sz[n++] = (size_t)n_opts * 4;                           // 11 opt_devs
  sz[n++] = (size_t)(n_meshes + 1) * 4;                   // 12 opt_off
  sz[n++] = (size_t)2 * n_meshes * (L + 1) * 8;           // 13 cb_same|cb_next
  sz[n++] = (size_t)(G + 1) * 4;                          // 14 g_mesh
  sz[n++] = (size_t)(G + 1) * 4;                          // 15 g_avail
  sz[n++] = (size_t)(G + 1) * 4;                          // 16 g_crow
  sz[n++] = (y.rows + 1) * 4;                             // 17 span_off
  sz[n++] = y.nnz_cap * 4;                                // 18 span_items
  sz[n++] = y.nnz_cap * sizeof(hapt_span);                // 19 spans
  sz[n++] = y.nnz_cap * 4;                                // 20 span_srank
  sz[n++] = y.pool_cap * 8;                               // 21 pool
  sz[n++] = 16 * 8;                                       // 22 counters
  sz[n++] = y.rows * 2;                                   // 23 row_kmin
  // scratch
  sz[n++] = (size_t)3 * (L + 1) * 8;                      // 24 prefix sums
  sz[n++] = (size_t)(L + 2) * (L + 2) * 4;                // 25 lcp
  sz[n++] = (y.rows + 1) * 4;                             // 26 row counts
  sz[n++] = y.nnz_cap * 8;                                // 27 keys a
  sz[n++] = y.nnz_cap * 8;                                // 28 keys b
  sz[n++] = (y.pool_cap + 1) * 8;                         // 29 rank histogram / scan
  sz[n++] = kCubTempBase + y.nnz_cap * 16;                // 30 cub temp
  sz[n++] = y.rows * (size_t)(L + 2) * 2;                 // 31 row_pos (table, after scratch)
  size_t cur = 0;
  for (int i = 0; i < n; ++i) {
    y.off[i] = cur;
    cur += align_up(sz[i]);
  }
  y.total = cur;
  return y;
}

struct Scratch {
  double *prefix;
  int32_t *lcp;
  int32_t *row_cnt;
  unsigned long long *keys_a, *keys_b;
  long long *hist;
  void *cub_temp;
  size_t cub_bytes;
};

Scratch scratch_of(const hapt_tables *t) {
  Layout y = layout(t->L, t->G, t->n_opts, t->n_meshes);
  char *base = (char *)t->t_tab;  // buffer start
  Scratch s;
  s.prefix = (double *)(base + y.off[24]);
  s.lcp = (int32_t *)(base + y.off[25]);
  s.row_cnt = (int32_t *)(base + y.off[26]);
  s.keys_a = (unsigned long long *)(base + y.off[27]);
  s.keys_b = (unsigned long long *)(base + y.off[28]);
  s.hist = (long long *)(base + y.off[29]);
  s.cub_temp = base + y.off[30];
  s.cub_bytes = kCubTempBase + y.nnz_cap * 16;
  return s;
}

// ---- K1a: option / budget metadata, prefix sums, boundary costs ----------
// opt_* and g_* : DpTables.__init__ (planner.py:179-226)
// prefix sums   : ProfileStore._build (profiling.py:218-224), sequential fp64
// cb_same/next  : boundary_costs (profiling.py:128-147) gathered as
//                 DpTables.cb_same/cb_next (planner.py:203-211)
__global__ void k1_meta(hapt_tables t, hapt_model_desc d, double *prefix) {
  const int L = d.L, nm = d.n_meshes, no = d.n_opts;
  for (int o = threadIdx.x; o < no; o += blockDim.x) {
    const int m = d.opt_mesh[o];
    t.opt_mesh[o] = m;
    t.opt_devs[o] = d.opt_n[o] * d.opt_m[o];
    t.opt_cap[o] = d.mesh_mem[m];
  }
  if (threadIdx.x == 0) {
    t.opt_off[0] = 0;
    for (int m = 0; m < nm; ++m) {
      int c = 0;
      for (int o = 0; o < no; ++o) c += (d.opt_mesh[o] == m);
      t.opt_off[m + 1] = t.opt_off[m] + c;
    }
    // remaining-device scalar g -> (mesh being consumed, devices left in it)
    int suffix_next = 0;  // suffix[m+1]
    t.g_mesh[0] = 0;
    t.g_avail[0] = 0;
    for (int m = nm - 1; m >= 0; --m) {
      const int budget = d.mesh_hosts[m] * d.mesh_dph[m];
      for (int g = suffix_next + 1; g <= suffix_next + budget; ++g) {
        t.g_mesh[g] = m;
        t.g_avail[g] = g - suffix_next;
      }
      suffix_next += budget;
    }
  }
  if (threadIdx.x == 32) {
    double f = 0.0, p = 0.0, a = 0.0;
    prefix[0] = 0.0;
    prefix[L + 1] = 0.0;
    prefix[2 * (L + 1)] = 0.0;
    for (int i = 1; i <= L; ++i) {
      f = __dadd_rn(f, d.layer_flops[i - 1]);
      p = __dadd_rn(p, d.layer_params[i - 1]);
      a = __dadd_rn(a, d.layer_bbytes[i - 1]);
      prefix[i] = f;
      prefix[(L + 1) + i] = p;
      prefix[2 * (L + 1) + i] = a;
    }
  }
  for (int x = threadIdx.x; x < nm * (L + 1); x += blockDim.x) {
    const int m = x / (L + 1), i = x % (L + 1);
    double same = 0.0, next = 0.0;
    if (i >= 1 && i < L) {
      const double bytes = d.layer_bbytes[i - 1];
      same = __ddiv_rn(bytes, d.mesh_inter_bw[m]);
      if (m + 1 < nm) next = __dadd_rn(__ddiv_rn(bytes, d.cross_bw_next[m]), d.cross_latency);
    }
    t.cb_same[x] = same;
    t.cb_next[x] = next;
  }
}

// ---- K1b: signature longest-common-prefix along each diagonal -------------
// lcp[a][b] (a <= b): number of equal layer signatures starting at a and b.
__global__ void k1_lcp(const int32_t *sig, int L, int32_t *lcp) {
  const int dgn = blockIdx.x * blockDim.x + threadIdx.x;  // b - a
  if (dgn >= L) return;
  int run = 0;
  for (int a = L - dgn; a >= 1; --a) {
    const int b = a + dgn;
    run = (sig[a - 1] == sig[b - 1]) ? run + 1 : 0;
    lcp[a * (L + 2) + b] = run;
  }
}

// canon_q[q][p]: start of the first span (q-major order) whose signature key
// equals that of [q,p] -- the canonical entry of profiling.py:241-251.
__global__ void k1_canon(int L, int dedup, const int32_t *lcp, int32_t *canon) {
  const long x = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= (long)(L + 2) * (L + 2)) return;
  const int q = (int)(x / (L + 2)), p = (int)(x % (L + 2));
  if (q < 1 || q > L || p < q || p > L) {
    canon[x] = 0;
    return;
  }
  int c = q;
  if (dedup) {
    // first a < q with lcp >= len, eight independent loads per step
    const int len = p - q + 1;
    for (int a0 = 1; a0 < q && c == q; a0 += 8) {
      int v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = a0 + u < q ? lcp[(a0 + u) * (L + 2) + q] : -1;
#pragma unroll
      for (int u = 7; u >= 0; --u)
        if (v[u] >= len) c = a0 + u;
    }
  }
  canon[x] = c;
}

// ---- K1c: analytic profile + OOM / imbalance masks, one thread per cell ----
__global__ void k1_profile(hapt_tables t, hapt_model_desc d, const double *prefix) {
  __shared__ unsigned long long st[6];
  if (threadIdx.x < 6) st[threadIdx.x] = 0;
  __syncthreads();
  const int L = d.L, S = L + 2;
  const long x = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long cells = (long)d.n_opts * S * S;
  if (x < cells) {
    const int o = (int)(x / ((long)S * S));
    const int q = (int)((x / S) % S);
    const int p = (int)(x % S);
    double t_tab = kInf, mp_tab = kInf, ma_tab = kInf;
    double tf = 0.0, tb = 0.0, mp = 0.0, ma = 0.0;
    int state = 0;
    if (q >= 1 && q <= L && p >= q && p <= L) {
      const int qc = t.canon_q[q * S + p];
      const int pc = qc + (p - q);
      const double *pf = prefix, *pp = prefix + (L + 1), *pa = prefix + 2 * (L + 1);
      // StageCandidate of the canonical span (profiling.py:229-236)
      const double flops = __dsub_rn(pf[pc], pf[qc - 1]);
      const double params = __dsub_rn(pp[pc], pp[qc - 1]);
      const double act = __dsub_rn(pa[pc], pa[qc - 1]);
      const int m = d.opt_mesh[o];
      const int sn = d.opt_n[o];
      const int devs = sn * d.opt_m[o];
      const double peak = d.mesh_peak[m];
      // analytic_profile (profiling.py:95-102)
      tf = __ddiv_rn(flops, __dmul_rn(__dmul_rn((double)devs, peak), d.efficiency));
      if (devs > 1 && d.alpha > 0.0) {
        const double link = (sn == 1) ? d.mesh_intra_bw[m] : d.mesh_inter_bw[m];
        tf = __dadd_rn(tf, __ddiv_rn(__dmul_rn(d.alpha, act), link));
      }
      tb = __dmul_rn(d.beta, tf);
      mp = __ddiv_rn(__dmul_rn(params, d.replication), (double)devs);
      ma = __ddiv_rn(__dmul_rn(d.act_factor, act), (double)devs);
      // pruning on the canonical profile (profiling.py:238, 253-275)
      const double fshare = (d.total_flops > 0.0) ? __ddiv_rn(flops, d.total_flops) : 0.0;
      const double cshare = __ddiv_rn(__dmul_rn((double)devs, peak), d.total_peak);
      const double need = __dadd_rn(mp, ma);
      int reason = 0;
      const double rho = d.imbalance_ratio;
      if (need > d.mesh_mem[m]) {
        reason = 1;
      } else if (isfinite(rho) && fshare > 0.0 &&
                 (fshare > __dmul_rn(rho, cshare) || cshare > __dmul_rn(rho, fshare))) {
        reason = 2;
      }
      const bool canonical = (qc == q);
      const bool feasible = (reason == 0);
      // measured overrides replace the canonical entry (profiling.py:353-366)
      if (d.ovr_index) {
        const int oi = d.ovr_index[((long)o * S + qc) * S + pc];
        if (oi >= 0) {
          tf = d.ovr_vals[4 * oi + 0];
          tb = d.ovr_vals[4 * oi + 1];
          mp = d.ovr_vals[4 * oi + 2];
          ma = d.ovr_vals[4 * oi + 3];
        }
      }
      if (feasible) {
        t_tab = __dadd_rn(tf, tb);  // StageMeshProfile.t (profiling.py:84-85)
        mp_tab = mp;
        ma_tab = ma;
      }
      state = (feasible ? 1 : 0) | (canonical ? 2 : 0) | (reason << 2);
      atomicAdd(&st[0], 1ull);
      if (canonical) atomicAdd(&st[1], 1ull);
      if (canonical && feasible) atomicAdd(&st[2], 1ull);
      if (!canonical) atomicAdd(&st[3], 1ull);
      if (reason == 1) atomicAdd(&st[4], 1ull);
      if (reason == 2) atomicAdd(&st[5], 1ull);
    }
    t.t_tab[x] = t_tab;
    t.mp_tab[x] = mp_tab;
    t.ma_tab[x] = ma_tab;
    t.tf_raw[x] = tf;
    t.tb_raw[x] = tb;
    t.mp_raw[x] = mp;
    t.ma_raw[x] = ma;
    t.cell_state[x] = (int8_t)state;
  }
  __syncthreads();
  if (threadIdx.x < 6 && st[threadIdx.x])
    atomicAdd((unsigned long long *)&t.counters[2 + threadIdx.x], st[threadIdx.x]);
}

// ---- CSR feasible-span index (planner.py:229-241) --------------------------
__global__ void k_row_count(hapt_tables t, int32_t *row_cnt) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int L = t.L, S = L + 2;
  const long rows = (long)t.n_opts * S;
  if (r > rows) return;
  if (r == rows) {
    row_cnt[r] = 0;
    return;
  }
  const int k = (int)(r % S);
  int c = 0;
  if (k >= 1 && k <= L) {
    const double *row = t.t_tab + r * S;
    for (int p = k; p <= L; ++p) c += isfinite(row[p]) ? 1 : 0;
  }
  row_cnt[r] = c;
}

__global__ void k_row_fill(hapt_tables t) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int L = t.L, S = L + 2;
  if (r >= (long)t.n_opts * S) return;
  const int k = (int)(r % S);
  if (k < 1 || k > L) return;
  const double *row = t.t_tab + r * S;
  int w = t.span_off[r];
  for (int p = k; p <= L; ++p)
    if (isfinite(row[p])) t.span_items[w++] = p;
}

// ---- finalize: per-entry DP metadata + the t_max pool ----------------------
__global__ void k_fill_keys(unsigned long long *keys, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) keys[i] = kPadKey;
}

// One thread per CSR entry (the memory threshold is a 16-step binary search,
// so a thread per row serialised up to L of them); the entry's row is found
// by binary search over span_off.
__global__ void k_span_meta(hapt_tables t, unsigned long long *keys) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int L = t.L, S = L + 2;
  const long rows = (long)t.n_opts * S;
  if (idx >= t.span_off[rows]) return;
  long lo = 0, hi = rows;  // last row with span_off[row] <= idx
  while (hi - lo > 1) {
    const long mid = (lo + hi) >> 1;
    if (t.span_off[mid] <= idx) lo = mid; else hi = mid;
  }
  const long r = lo;
  const int o = (int)(r / S);
  const int p = t.span_items[idx];
  const double tt = t.t_tab[r * S + p];
  hapt_span sp;
  sp.tt = tt;
  sp.prank = 0;
  sp.i = (uint16_t)p;
  sp.kmax = (uint16_t)mem_kmax(t.mp_tab[r * S + p], t.ma_tab[r * S + p], t.opt_cap[o]);
  t.spans[idx] = sp;
  keys[idx] = isfinite(tt) ? fkey(tt) : kPadKey;
}

__global__ void k_row_kmin(hapt_tables t) {
  const long r = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (long)t.n_opts * (t.L + 2)) return;
  int kmin = kKSat;
  for (int idx = t.span_off[r]; idx < t.span_off[r + 1]; ++idx) kmin = min(kmin, (int)t.spans[idx].kmax);
  t.row_kmin[r] = (uint16_t)kmin;
}

__global__ void k_pool_decode(hapt_tables t, const unsigned long long *uniq,
                              const long long *num_unique) {
  const long nu = *num_unique;
  const long plen = (nu > 0 && uniq[nu - 1] == kPadKey) ? nu - 1 : nu;
  const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) t.counters[1] = plen;
  if (i < plen) t.pool[i] = fdecode(uniq[i]);
}

__device__ __forceinline__ int lower_bound(const double *a, int n, double v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_prank(hapt_tables t) {
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const long nnz = t.span_off[(long)t.n_opts * (t.L + 2)];
  if (idx == 0) t.counters[0] = nnz;
  if (idx >= nnz) return;
  const double tt = t.spans[idx].tt;
  // entries with a non-finite t can never win a cell in the reference
  // (tt > t_max, or cand = NaN/inf never < best), so they get rank INT_MAX
  t.spans[idx].prank = isfinite(tt) ? lower_bound(t.pool, (int)t.counters[1], tt) : 0x7fffffff;
}

// Row suffix-min pool ranks and the per-row position table row_pos[row][i]
// = #entries with span end <= i (entries are in ascending span end).
// One warp per row (a thread per row walked up to L entries twice, one
// dependent load at a time): suffix minimum of the pool ranks from the row's
// end in 32-entry chunks, then row_pos[i] = #entries with span end <= i by a
// binary search per i (entries are in ascending span end).
__global__ void k_srank(hapt_tables t) {
  const long r = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int S = t.L + 2;
  if (r >= (long)t.n_opts * S) return;  // warp-uniform
  const int beg = t.span_off[r], end = t.span_off[r + 1];
  int carry = 0x7fffffff;
  for (int c1 = end; c1 > beg; c1 -= 32) {  // chunk [c1-32, c1)
    const int idx = c1 - 32 + lane;
    int m = idx >= beg ? t.spans[idx].prank : 0x7fffffff;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_down_sync(0xffffffffu, m, off);
      if (lane + off < 32) m = min(m, y);
    }
    m = min(m, carry);
    if (idx >= beg) t.span_srank[idx] = m;
    carry = __shfl_sync(0xffffffffu, m, 0);
  }
  uint16_t *pos = t.row_pos + r * S;
  for (int i = lane; i < S; i += 32) {
    int lo = beg, hi = end;  // first entry with span end > i
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)t.spans[mid].i <= i) lo = mid + 1; else hi = mid;
    }
    pos[i] = (uint16_t)(lo - beg);
  }
}

// Boundary row a state g reads when it is the successor of a new first stage
// (derivation in DESIGN.md §K2).  A caller g' > g in mesh r reaches g with
// g >= g' - g_avail[g'], so: g strictly inside mesh r (g_mesh[g+1] == g_mesh[g])
// -> same mesh, cb_same[r]; g the full budget of its mesh, or g = 0 -> the
// caller left mesh r = g_mesh[g+1] -> cb_next[r]; g = G has no caller.
//
// Stated for any (g_mesh, g_avail) encoding a drop-in caller may pass
// (_dp.pyx:58-77): every caller g > g2 whose mesh r = g_mesh[g] has an option
// of exactly g - g2 <= g_avail[g] devices reads cb_same[r] if g2 >= 1 and
// g_mesh[g2] == r, else cb_next[r].  The DP hoists c into the successor
// table, so the row must not depend on the caller; DpTables' encoding
// (meshes consumed in order) always satisfies this and gives the rule above.
// A state with callers that disagree raises counters[10] (the host refuses
// the encoding); a state with no caller gets -1 (its entry is never read).
__global__ void k_gcrow(hapt_tables t) {
  // one warp per successor state g2, lanes over the callers g
  const int g2 = (int)(((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (g2 > t.G) return;  // warp-uniform
  const int nm = t.n_meshes;
  int lo = 0x7fffffff, hi = -1;
  bool conflict = false;
  for (int g = g2 + 1 + lane; g <= t.G; g += 32) {
    const int r = t.g_mesh[g], devs = g - g2;
    if (r < 0 || r >= nm) {
      conflict = true;
      continue;
    }
    if (devs > t.g_avail[g]) continue;
    bool has = false;
    for (int o = t.opt_off[r]; o < t.opt_off[r + 1] && !has; ++o) has = t.opt_devs[o] == devs;
    if (!has) continue;
    const int rr = (g2 >= 1 && t.g_mesh[g2] == r) ? r : nm + r;
    lo = min(lo, rr);
    hi = max(hi, rr);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  conflict = __any_sync(0xffffffffu, conflict) || (hi >= 0 && lo != hi);
  if (lane == 0) {
    t.g_crow[g2] = hi;  // -1: no caller
    if (conflict) t.counters[10] = 1;
  }
}

// Encoding checks the DP relies on besides g_crow: every option uses at least
// one device (cells with fewer devices than remaining stages are skipped).
__global__ void k_encoding(hapt_tables t) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o < t.n_opts && t.opt_devs[o] < 1) t.counters[10] = 1;
}

}  // namespace

void *tables_hist(const hapt_tables *t) { return scratch_of(t).hist; }

int finalize_impl(hapt_tables *tp, cudaStream_t st) {
  hapt_tables &t = *tp;
  Scratch s = scratch_of(&t);
  Layout y = layout(t.L, t.G, t.n_opts, t.n_meshes);
  const size_t rows = y.rows;
  k_fill_keys<<<grid_for(y.nnz_cap, 256), 256, 0, st>>>(s.keys_a, y.nnz_cap); ::hapt::note_launch();
  k_span_meta<<<grid_for(y.nnz_cap, 128), 128, 0, st>>>(t, s.keys_a); ::hapt::note_launch();
  k_row_kmin<<<grid_for(rows, 128), 128, 0, st>>>(t); ::hapt::note_launch();
  HAPT_LAUNCHED("k_span_meta");
  cub::DoubleBuffer<unsigned long long> db(s.keys_a, s.keys_b);
  size_t need = 0;
  HAPT_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, need, db, (int)y.nnz_cap, 0, 64, st));
  if (need > s.cub_bytes) {
    set_error("cub radix-sort temp %zu > %zu", need, s.cub_bytes);
    return HAPT_ENOSPACE;
  }
  HAPT_CUDA(cub::DeviceRadixSort::SortKeys(s.cub_temp, need, db, (int)y.nnz_cap, 0, 64, st));
  unsigned long long *sorted = db.Current();
  unsigned long long *uniq = db.Alternate();
  long long *num_unique = (long long *)&t.counters[8];
  need = 0;
  HAPT_CUDA(cub::DeviceSelect::Unique(nullptr, need, sorted, uniq, num_unique, (int)y.nnz_cap, st));
  if (need > s.cub_bytes) {
    set_error("cub unique temp %zu > %zu", need, s.cub_bytes);
    return HAPT_ENOSPACE;
  }
  HAPT_CUDA(cub::DeviceSelect::Unique(s.cub_temp, need, sorted, uniq, num_unique, (int)y.nnz_cap, st));
  k_pool_decode<<<grid_for(y.pool_cap, 256), 256, 0, st>>>(t, uniq, num_unique); ::hapt::note_launch();
  k_prank<<<grid_for(y.nnz_cap, 256), 256, 0, st>>>(t); ::hapt::note_launch();
  k_srank<<<grid_for(rows * 32, 256), 256, 0, st>>>(t); ::hapt::note_launch();
  HAPT_CUDA(cudaMemsetAsync(&t.counters[10], 0, 8, st));
  k_encoding<<<grid_for(t.n_opts, 128), 128, 0, st>>>(t); ::hapt::note_launch();
  k_gcrow<<<grid_for((size_t)(t.G + 1) * 32, 128), 128, 0, st>>>(t); ::hapt::note_launch();
  HAPT_LAUNCHED("finalize");
  return HAPT_OK;
}

}  // namespace hapt

using namespace hapt;

extern "C" size_t hapt_tables_bytes(int32_t L, int32_t G, int32_t n_opts, int32_t n_meshes) {
  return layout(L, G, n_opts, n_meshes).total;
}

extern "C" int hapt_tables_init(hapt_tables *t, void *buf, size_t buf_bytes, int32_t L,
                                int32_t G, int32_t n_opts, int32_t n_meshes) {
  if (!t || !buf || L < 1 || G < 1 || n_opts < 1 || n_meshes < 1) {
    set_error("hapt_tables_init: invalid dimensions");
    return HAPT_EINVAL;
  }
  if (L >= 4095) {  // 16-bit span index; the DP's multiply-high cell decode needs L < 2^12
    set_error("hapt_tables_init: L=%d exceeds the supported 4094 layers", L);
    return HAPT_EINVAL;
  }
  Layout y = layout(L, G, n_opts, n_meshes);
  if (buf_bytes < y.total) {
    set_error("hapt_tables_init: buffer %zu < %zu", buf_bytes, y.total);
    return HAPT_ENOSPACE;
  }
  if (((uintptr_t)buf) % 256) {
    set_error("hapt_tables_init: buffer must be 256-byte aligned");
    return HAPT_EINVAL;
  }
  char *b = (char *)buf;
  t->L = L;
  t->G = G;
  t->n_opts = n_opts;
  t->n_meshes = n_meshes;
  t->s_max = L < G ? L : G;
  // (G+1)(L+1) successor slots: a slot's byte offset (x 1 KB at 4 candidates
  // per lane) is a 32-bit word of the staged transition, and the dense-layer
  // cell decode is exact below 2^20 cells; n_opts: the per-option shared
  // arrays of dp_prep; the CSR index itself is int32 (nnz < 2^31).
  if ((size_t)(G + 1) * (L + 1) >= (1u << 20) || n_opts >= 2048 ||
      (size_t)n_opts * L * (L + 1) / 2 >= (1ull << 31)) {
    set_error("hapt_tables_init: (G+1)(L+1)=%zu, n_opts=%d or the span count exceeds the "
              "supported range", (size_t)(G + 1) * (L + 1), n_opts);
    return HAPT_EINVAL;
  }
  if (3 * t->s_max + 3 >= kKSat) {
    set_error("hapt_tables_init: s_max=%d too large for 16-bit launch bounds", t->s_max);
    return HAPT_EINVAL;
  }
  t->nnz_cap = (int32_t)y.nnz_cap;
  t->pool_cap = (int32_t)y.pool_cap;
  t->t_tab = (double *)(b + y.off[0]);
  t->mp_tab = (double *)(b + y.off[1]);
  t->ma_tab = (double *)(b + y.off[2]);
  t->tf_raw = (double *)(b + y.off[3]);
  t->tb_raw = (double *)(b + y.off[4]);
  t->mp_raw = (double *)(b + y.off[5]);
  t->ma_raw = (double *)(b + y.off[6]);
  t->cell_state = (int8_t *)(b + y.off[7]);
  t->canon_q = (int32_t *)(b + y.off[8]);
  t->opt_cap = (double *)(b + y.off[9]);
  t->opt_mesh = (int32_t *)(b + y.off[10]);
  t->opt_devs = (int32_t *)(b + y.off[11]);
  t->opt_off = (int32_t *)(b + y.off[12]);
  t->cb_same = (double *)(b + y.off[13]);
  t->cb_next = t->cb_same + (size_t)n_meshes * (L + 1);
  t->g_mesh = (int32_t *)(b + y.off[14]);
  t->g_avail = (int32_t *)(b + y.off[15]);
  t->g_crow = (int32_t *)(b + y.off[16]);
  t->span_off = (int32_t *)(b + y.off[17]);
  t->span_items = (int32_t *)(b + y.off[18]);
  t->spans = (hapt_span *)(b + y.off[19]);
  t->span_srank = (int32_t *)(b + y.off[20]);
  t->pool = (double *)(b + y.off[21]);
  t->counters = (int64_t *)(b + y.off[22]);
  t->row_kmin = (uint16_t *)(b + y.off[23]);
  t->row_pos = (uint16_t *)(b + y.off[31]);
  t->scratch = b + y.off[24];
  t->scratch_bytes = y.off[31] - y.off[24];
  return HAPT_OK;
}

extern "C" int hapt_tables_build(hapt_tables *t, const hapt_model_desc *d, void *stream) {
  if (!t || !d || d->L != t->L || d->G != t->G || d->n_opts != t->n_opts ||
      d->n_meshes != t->n_meshes) {
    set_error("hapt_tables_build: description does not match the tables");
    return HAPT_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch s = scratch_of(t);
  Layout y = layout(t->L, t->G, t->n_opts, t->n_meshes);
  const int L = t->L;
  HAPT_CUDA(cudaMemsetAsync(t->counters, 0, 16 * 8, st));
  HAPT_CUDA(cudaMemsetAsync(s.lcp, 0, (size_t)(L + 2) * (L + 2) * 4, st));
  k1_meta<<<1, 256, 0, st>>>(*t, *d, s.prefix); ::hapt::note_launch();
  k1_lcp<<<grid_for(L, 128), 128, 0, st>>>(d->layer_sig, L, s.lcp); ::hapt::note_launch();
  k1_canon<<<grid_for((size_t)(L + 2) * (L + 2), 256), 256, 0, st>>>(L, d->dedup, s.lcp, t->canon_q); ::hapt::note_launch();
  k1_profile<<<grid_for(y.cells, 256), 256, 0, st>>>(*t, *d, s.prefix); ::hapt::note_launch();
  HAPT_LAUNCHED("k1_profile");
  k_row_count<<<grid_for(y.rows + 1, 128), 128, 0, st>>>(*t, s.row_cnt); ::hapt::note_launch();
  size_t need = 0;
  HAPT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, s.row_cnt, t->span_off, (int)(y.rows + 1), st));
  if (need > s.cub_bytes) {
    set_error("cub scan temp %zu > %zu", need, s.cub_bytes);
    return HAPT_ENOSPACE;
  }
  HAPT_CUDA(cub::DeviceScan::ExclusiveSum(s.cub_temp, need, s.row_cnt, t->span_off, (int)(y.rows + 1), st));
  k_row_fill<<<grid_for(y.rows, 128), 128, 0, st>>>(*t); ::hapt::note_launch();
  HAPT_LAUNCHED("k_row_fill");
  return finalize_impl(t, st);
}

extern "C" int hapt_tables_finalize(hapt_tables *t, void *stream) {
  if (!t) {
    set_error("hapt_tables_finalize: null tables");
    return HAPT_EINVAL;
  }
  return finalize_impl(t, (cudaStream_t)stream);
}
