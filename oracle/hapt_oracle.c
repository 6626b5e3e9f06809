/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Never linked into, imported by, or
 * called from the product path (paper_2509_24859_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker / CPU baseline.
 *
 * Plain-C restatement of the reference algorithms of the planner hot path
 * (meshpipe, arXiv 2509.24859 planner; files under /root/reference/pkg/src/
 * meshpipe/).  Pinned against golden vectors produced by the reference
 * itself (tests/golden/, tests/test_oracle.py).
 *
 * Built with -O2 -ffp-contract=off (no FMA: the reference's Cython build has
 * none).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------
 * Stage-partition DP for one t_max -- _dp.pyx:38-95 (and dp_py.py:44-102).
 * Arrays are C-contiguous with the DpTables shapes (planner.py:164-248).
 * ---------------------------------------------------------------------- */
void oracle_dp_sweep(double t_max, const double *t_tab, const double *mp_tab,
                     const double *ma_tab, const double *opt_cap, const int32_t *opt_mesh,
                     const int32_t *opt_devs, const int32_t *opt_off,
                     const double *cb_same, const double *cb_next, const int32_t *g_mesh,
                     const int32_t *g_avail, int32_t s_max, const int32_t *span_off,
                     const int32_t *span_items, int32_t L, int32_t G, double *F, double *N,
                     int32_t *bp_i, int32_t *bp_o) {
  (void)opt_mesh;
  const long stride = L + 2;
  const long plane = (long)(L + 2) * (G + 1);
  const long total = (long)(s_max + 1) * plane;
  for (long x = 0; x < total; ++x) {
    F[x] = INFINITY;
    N[x] = 0.0;
    bp_i[x] = -1;
    bp_o[x] = -1;
  }
#define AT(s, k, g) ((long)(s) * plane + (long)(k) * (G + 1) + (g))
  F[AT(0, L + 1, 0)] = 0.0; /* _dp.pyx:41 */
  for (int s = 1; s <= s_max; ++s) {
    for (int k = L; k >= 1; --k) {
      for (int g = 1; g <= G; ++g) {
        const int r = g_mesh[g], avail = g_avail[g];
        double best = INFINITY, best_n = 0.0;
        int best_i = -1, best_o = -1;
        for (int o = opt_off[r]; o < opt_off[r + 1]; ++o) {
          const int devs = opt_devs[o];
          if (devs > avail) continue;
          const int g2 = g - devs;
          const int same = (g2 >= 1) && (g_mesh[g2] == r);
          for (int idx = span_off[o * stride + k]; idx < span_off[o * stride + k + 1]; ++idx) {
            const int i = span_items[idx];
            const double fc = F[AT(s - 1, i + 1, g2)];
            if (fc == INFINITY) continue;
            const double c = same ? cb_same[(long)r * (L + 1) + i] : cb_next[(long)r * (L + 1) + i];
            if (c > t_max) continue;
            const long cell = ((long)o * stride + k) * stride + i;
            const double tt = t_tab[cell];
            if (tt > t_max) continue;
            /* _dp.pyx:82-84, same association */
            const double kk = ceil(2.0 * c / t_max) + 1.0 + N[AT(s - 1, i + 1, g2)];
            if (mp_tab[cell] + kk * ma_tab[cell] > opt_cap[o]) continue;
            const double cand = tt + (2.0 * c + fc);
            if (cand < best) {
              best = cand;
              best_n = kk;
              best_i = i;
              best_o = o;
            }
          }
        }
        if (best_i >= 0) {
          F[AT(s, k, g)] = best;
          N[AT(s, k, g)] = best_n;
          bp_i[AT(s, k, g)] = best_i;
          bp_o[AT(s, k, g)] = best_o;
        }
      }
    }
  }
#undef AT
}

/* ------------------------------------------------------------------------
 * ProfileStore._build + analytic_profile (profiling.py:88-103, 212-286),
 * materialised as DpTables dense tables (planner.py:191-201).
 * Dedup: the canonical entry of a span is the first span in q-major order
 * with an equal layer-signature sequence, found here by direct comparison
 * (the kernel uses an LCP table; the oracle deliberately does not).
 * Outputs [n_opts][L+2][L+2]: t (inf if infeasible), tf, tb, mp, ma (raw
 * profile values), state (bit0 feasible, bit1 canonical, bits2-3 reason);
 * stats[6] = StoreStats.
 * ---------------------------------------------------------------------- */
void oracle_profile(int32_t L, const double *flops, const double *params, const double *bbytes,
                    const int32_t *sig, int32_t n_opts, const int32_t *opt_mesh,
                    const int32_t *opt_n, const int32_t *opt_m, const double *mesh_peak,
                    const double *mesh_mem, const double *mesh_intra, const double *mesh_inter,
                    double beta, double eff, double alpha, double repl, double act_factor,
                    double rho, double total_flops, double total_peak, int32_t dedup,
                    double *t_out, double *tf_out, double *tb_out, double *mp_out,
                    double *ma_out, int8_t *state_out, int64_t *stats) {
  const long S = L + 2;
  double *pf = calloc(L + 1, sizeof(double));
  double *pp = calloc(L + 1, sizeof(double));
  double *pa = calloc(L + 1, sizeof(double));
  for (int i = 1; i <= L; ++i) { /* profiling.py:218-224 */
    pf[i] = pf[i - 1] + flops[i - 1];
    pp[i] = pp[i - 1] + params[i - 1];
    pa[i] = pa[i - 1] + bbytes[i - 1];
  }
  for (long x = 0; x < (long)n_opts * S * S; ++x) {
    t_out[x] = INFINITY;
    tf_out[x] = tb_out[x] = mp_out[x] = ma_out[x] = 0.0;
    state_out[x] = 0;
  }
  for (int j = 0; j < 6; ++j) stats[j] = 0;
  for (int q = 1; q <= L; ++q) {
    for (int p = q; p <= L; ++p) {
      const int len = p - q + 1;
      int qc = q;
      if (dedup) {
        for (int a = 1; a < q; ++a) {
          int eq = 1;
          for (int j = 0; j < len && eq; ++j) eq = (sig[a - 1 + j] == sig[q - 1 + j]);
          if (eq) {
            qc = a;
            break;
          }
        }
      }
      const int pc = qc + len - 1;
      const double cf = pf[pc] - pf[qc - 1];
      const double cp = pp[pc] - pp[qc - 1];
      const double ca = pa[pc] - pa[qc - 1];
      for (int o = 0; o < n_opts; ++o) {
        const int m = opt_mesh[o], devs = opt_n[o] * opt_m[o];
        double t_f = cf / ((devs * mesh_peak[m]) * eff);
        if (devs > 1 && alpha > 0.0) {
          const double link = opt_n[o] == 1 ? mesh_intra[m] : mesh_inter[m];
          t_f += alpha * ca / link;
        }
        const double t_b = beta * t_f;
        const double mem_p = cp * repl / devs;
        const double mem_a = act_factor * ca / devs;
        const double fshare = total_flops > 0 ? cf / total_flops : 0.0;
        const double cshare = devs * mesh_peak[m] / total_peak;
        int reason = 0;
        if (mem_p + mem_a > mesh_mem[m]) reason = 1;
        else if (isfinite(rho) && fshare > 0 && (fshare > rho * cshare || cshare > rho * fshare))
          reason = 2;
        const int canonical = (qc == q);
        const long x = ((long)o * S + q) * S + p;
        tf_out[x] = t_f;
        tb_out[x] = t_b;
        mp_out[x] = mem_p;
        ma_out[x] = mem_a;
        if (!reason) t_out[x] = t_f + t_b;
        state_out[x] = (int8_t)((reason == 0) | (canonical << 1) | (reason << 2));
        stats[0] += 1;
        stats[1] += canonical;
        stats[2] += canonical && !reason;
        stats[3] += !canonical;
        stats[4] += reason == 1;
        stats[5] += reason == 2;
      }
    }
  }
  free(pf);
  free(pp);
  free(pa);
}

/* ------------------------------------------------------------------------
 * build_dag + simulate (simulation.py:73-149, 204-228): explicit DAG and a
 * Kahn sweep, for ONE plan.  Node numbering as the reference.  Returns the
 * number of processed nodes (== n_nodes unless the program deadlocks).
 * ---------------------------------------------------------------------- */
static long node_fb(int kind, int mb, int s, int B) { return 2L * ((long)(s - 1) * B + (mb - 1)) + kind; }
static long node_c(int kind, int mb, int s, int S, int B) {
  return 2L * S * B + 2L * ((long)(s - 1) * B + (mb - 1)) + kind;
}

long oracle_simulate(int32_t S, int32_t B, const double *t_fwd, const double *t_bwd,
                     const double *comm, const int32_t *counts, double *start, double *end,
                     double *makespan) {
  const long n = (long)B * (4L * S - 2) + 1;
  const long sink = n - 1;
  double *dur = malloc(n * sizeof(double));
  for (int s = 1; s <= S; ++s)
    for (int i = 1; i <= B; ++i) {
      dur[node_fb(0, i, s, B)] = t_fwd[s - 1];
      dur[node_fb(1, i, s, B)] = t_bwd[s - 1];
    }
  for (int s = 1; s < S; ++s)
    for (int i = 1; i <= B; ++i) {
      dur[node_c(0, i, s, S, B)] = comm[s - 1];
      dur[node_c(1, i, s, S, B)] = comm[s - 1];
    }
  dur[sink] = 0.0;
  /* edges (u, v) */
  const long max_e = 4L * S * B + 8L * S * B + n + 16;
  long *eu = malloc(max_e * sizeof(long)), *ev = malloc(max_e * sizeof(long));
  long ne = 0;
#define EDGE(a, b) do { eu[ne] = (a); ev[ne] = (b); ++ne; } while (0)
  for (int s = 1; s <= S; ++s) { /* program order, scheduling.py:241-249 */
    const int Nc = counts[s - 1];
    long prev = -1;
    for (int pos = 0; pos < 2 * B; ++pos) {
      int isF, mb;
      if (pos < Nc) {
        isF = 1;
        mb = pos + 1;
      } else if (pos - Nc < 2 * (B - Nc)) {
        const int q = pos - Nc;
        isF = q % 2;
        mb = isF ? Nc + (q + 1) / 2 : q / 2 + 1;
      } else {
        isF = 0;
        mb = (B - Nc) + (pos - Nc - 2 * (B - Nc)) + 1;
      }
      const long v = node_fb(isF ? 0 : 1, mb, s, B);
      if (prev >= 0) EDGE(prev, v);
      prev = v;
    }
  }
  for (int s = 1; s < S; ++s)
    for (int i = 1; i < B; ++i) {
      EDGE(node_c(0, i, s, S, B), node_c(0, i + 1, s, S, B));
      EDGE(node_c(1, i, s, S, B), node_c(1, i + 1, s, S, B));
    }
  for (int s = 1; s < S; ++s)
    for (int i = 1; i <= B; ++i) {
      EDGE(node_fb(0, i, s, B), node_c(0, i, s, S, B));
      EDGE(node_c(0, i, s, S, B), node_fb(0, i, s + 1, B));
      EDGE(node_fb(1, i, s + 1, B), node_c(1, i, s, S, B));
      EDGE(node_c(1, i, s, S, B), node_fb(1, i, s, B));
    }
  int *has_succ = calloc(n, sizeof(int));
  for (long e = 0; e < ne; ++e) has_succ[eu[e]] = 1;
  for (long v = 0; v < n - 1; ++v)
    if (!has_succ[v]) EDGE(v, sink);
#undef EDGE
  /* CSR of successors, Kahn sweep (simulation.py:207-223) */
  long *off = calloc(n + 1, sizeof(long)), *adj = malloc(ne * sizeof(long));
  long *indeg = calloc(n, sizeof(long)), *fill = calloc(n, sizeof(long));
  for (long e = 0; e < ne; ++e) {
    off[eu[e] + 1]++;
    indeg[ev[e]]++;
  }
  for (long v = 0; v < n; ++v) off[v + 1] += off[v];
  for (long e = 0; e < ne; ++e) adj[off[eu[e]] + fill[eu[e]]++] = ev[e];
  long *queue = malloc(n * sizeof(long));
  long head = 0, tail = 0;
  for (long v = 0; v < n; ++v) {
    start[v] = 0.0;
    if (indeg[v] == 0) queue[tail++] = v;
  }
  while (head < tail) {
    const long u = queue[head++];
    const double su_end = start[u] + dur[u];
    for (long x = off[u]; x < off[u + 1]; ++x) {
      const long v = adj[x];
      if (su_end > start[v]) start[v] = su_end;
      if (--indeg[v] == 0) queue[tail++] = v;
    }
  }
  double mk = 0.0;
  for (long v = 0; v < n; ++v) {
    end[v] = start[v] + dur[v];
    if (v == 0 || end[v] > mk) mk = end[v];
  }
  *makespan = mk;
  free(dur); free(eu); free(ev); free(has_succ); free(off); free(adj);
  free(indeg); free(fill); free(queue);
  return head;
}

/* adaptive_counts (scheduling.py:89-124) for one plan; returns 0, or the
 * 1-based boundary whose comm exceeds t_max (CommTooLargeError). */
int32_t oracle_adaptive_counts(int32_t S, const double *stage_t, const double *comm,
                               double epsilon, double t_max_override, int32_t *counts) {
  double tm = stage_t[0];
  for (int i = 1; i < S; ++i)
    if (stage_t[i] > tm) tm = stage_t[i];
  if (!isnan(t_max_override)) tm = t_max_override;
  counts[S - 1] = 1;
  for (int i = S - 2; i >= 0; --i) {
    const double c = comm[i];
    int d;
    if (c > tm) return i + 1;
    if (c <= epsilon * tm) d = 1;
    else if (c <= tm / 2) d = 2;
    else d = 3;
    counts[i] = counts[i + 1] + d;
  }
  return 0;
}

/* Config E batch (checker for the 10^5+-plan parity test): per plan p of
 * dense [P][8] inputs, adaptive counts with epsilon and t_max = max stage
 * time (scheduling.py:89-124), then the explicit-DAG makespan of
 * oracle_simulate (simulation.py:73-228).  status[p] = 0, or the boundary of
 * a CommTooLargeError.  Plans are independent, so `lo..hi` lets the caller
 * split the batch over host threads. */
void oracle_config_e_batch(int64_t lo, int64_t hi, int32_t B, const int32_t *S,
                           const double *t_fwd, const double *t_bwd, const double *comm,
                           double epsilon, int32_t *counts, int32_t *status, double *makespan) {
  long cap = 0;
  double *start = NULL, *end = NULL;
  for (int64_t p = lo; p < hi; ++p) {
    const int s = S[p];
    double st[8];
    for (int i = 0; i < s; ++i) st[i] = t_fwd[p * 8 + i] + t_bwd[p * 8 + i];
    status[p] = oracle_adaptive_counts(s, st, comm + p * 8, epsilon, NAN, counts + p * 8);
    makespan[p] = NAN;
    if (status[p]) continue;
    const long n = (long)B * (4L * s - 2) + 1;
    if (n > cap) {
      free(start);
      free(end);
      start = malloc(n * sizeof(double));
      end = malloc(n * sizeof(double));
      cap = n;
    }
    if (oracle_simulate(s, B, t_fwd + p * 8, t_bwd + p * 8, comm + p * 8, counts + p * 8, start,
                        end, makespan + p) != n)
      status[p] = -1; /* dependency cycle */
  }
  free(start);
  free(end);
}
