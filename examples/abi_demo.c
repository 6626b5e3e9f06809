/*
 * abi_demo.c -- the planner hot path driven from plain C through the C ABI
 * (include/hapt_b200.h): no Python, no torch.  What a non-Python host of the
 * reference (or a cgo / JNI binding) would call.
 *
 *   abi_demo <instance.txt>
 *
 * The instance file is whitespace-separated numbers (written by
 * tests/test_abi_demo.py from a golden instance):
 *   L n_meshes n_opts B
 *   layer_flops[L] layer_params[L] layer_bbytes[L] layer_sig[L]
 *   per mesh: hosts devices_per_host peak_flops mem_device intra_bw inter_bw
 *   cross_bw_next[n_meshes]
 *   opt_n[n_opts] opt_m[n_opts] opt_mesh[n_opts]
 *   cross_latency beta efficiency alpha replication act_factor rho
 *   total_flops total_peak dedup
 * Output (one line): t_max T* best_s n_stages then (start end option) per
 * stage -- the full-pool (T*, t_max) argmin, i.e. the reference search()'s
 * plan on the benchmark configs.
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hapt_b200.h"

#define CK(call)                                                              \
  do {                                                                        \
    int rc_ = (call);                                                         \
    if (rc_ != 0) {                                                           \
      fprintf(stderr, "%s failed: %d %s\n", #call, rc_, hapt_last_error());   \
      exit(1);                                                                \
    }                                                                         \
  } while (0)
#define CU(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));             \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

static void *dcopy(const void *h, size_t n) {
  void *d = NULL;
  CU(cudaMalloc(&d, n > 0 ? n : 1));
  if (n) CU(cudaMemcpy(d, h, n, cudaMemcpyHostToDevice));
  return d;
}

static void rd(FILE *f, double *x, int n) {
  for (int i = 0; i < n; ++i)
    if (fscanf(f, "%lf", &x[i]) != 1) exit(2);
}
static void ri(FILE *f, int32_t *x, int n) {
  for (int i = 0; i < n; ++i)
    if (fscanf(f, "%d", &x[i]) != 1) exit(2);
}

int main(int argc, char **argv) {
  if (argc < 2) return 2;
  FILE *f = fopen(argv[1], "r");
  if (!f) return 2;
  int32_t L, nm, no, B;
  if (fscanf(f, "%d %d %d %d", &L, &nm, &no, &B) != 4) return 2;
  double *fl = malloc(8 * L), *pa = malloc(8 * L), *bb = malloc(8 * L);
  int32_t *sig = malloc(4 * L);
  rd(f, fl, L), rd(f, pa, L), rd(f, bb, L), ri(f, sig, L);
  int32_t *hosts = malloc(4 * nm), *dph = malloc(4 * nm);
  double *peak = malloc(8 * nm), *mem = malloc(8 * nm), *intra = malloc(8 * nm),
         *inter = malloc(8 * nm), *cross = malloc(8 * nm);
  int32_t G = 0;
  for (int m = 0; m < nm; ++m) {
    double v[6];
    rd(f, v, 6);
    hosts[m] = (int32_t)v[0], dph[m] = (int32_t)v[1];
    peak[m] = v[2], mem[m] = v[3], intra[m] = v[4], inter[m] = v[5];
    G += hosts[m] * dph[m];
  }
  rd(f, cross, nm);
  int32_t *on = malloc(4 * no), *om = malloc(4 * no), *omesh = malloc(4 * no);
  ri(f, on, no), ri(f, om, no), ri(f, omesh, no);
  double sc[9];
  rd(f, sc, 9);
  int32_t dedup;
  if (fscanf(f, "%d", &dedup) != 1) return 2;
  fclose(f);

  hapt_model_desc d = {0};
  d.L = L, d.n_meshes = nm, d.n_opts = no, d.G = G;
  d.layer_flops = dcopy(fl, 8 * L), d.layer_params = dcopy(pa, 8 * L);
  d.layer_bbytes = dcopy(bb, 8 * L), d.layer_sig = dcopy(sig, 4 * L);
  d.mesh_hosts = dcopy(hosts, 4 * nm), d.mesh_dph = dcopy(dph, 4 * nm);
  d.mesh_peak = dcopy(peak, 8 * nm), d.mesh_mem = dcopy(mem, 8 * nm);
  d.mesh_intra_bw = dcopy(intra, 8 * nm), d.mesh_inter_bw = dcopy(inter, 8 * nm);
  d.cross_bw_next = dcopy(cross, 8 * nm);
  d.opt_n = dcopy(on, 4 * no), d.opt_m = dcopy(om, 4 * no), d.opt_mesh = dcopy(omesh, 4 * no);
  d.cross_latency = sc[0], d.beta = sc[1], d.efficiency = sc[2], d.alpha = sc[3];
  d.replication = sc[4], d.act_factor = sc[5], d.imbalance_ratio = sc[6];
  d.total_flops = sc[7], d.total_peak = sc[8], d.dedup = dedup;

  /* K1: tables in one caller-owned buffer */
  hapt_tables t;
  const size_t tb = hapt_tables_bytes(L, G, no, nm);
  void *tbuf = NULL;
  CU(cudaMalloc(&tbuf, tb));
  CK(hapt_tables_init(&t, tbuf, tb, L, G, no, nm));
  CK(hapt_tables_build(&t, &d, NULL));
  int64_t cnt[16];
  CU(cudaMemcpy(cnt, t.counters, sizeof(cnt), cudaMemcpyDeviceToHost));
  const int32_t pool = (int32_t)cnt[1];
  if (pool == 0) {
    printf("infeasible\n");
    return 0;
  }
  /* K2: every t_max candidate of the pool in one batch, then the argmin */
  const size_t ws_bytes = hapt_dp_workspace_bytes(&t, pool);
  void *ws = NULL;
  double *ftop = NULL, *tstar = NULL;
  int64_t *states = NULL;
  int32_t *best_s = NULL, *winner = NULL;
  CU(cudaMalloc(&ws, ws_bytes));
  CU(cudaMalloc((void **)&ftop, 8 * (size_t)pool * (t.s_max + 1)));
  CU(cudaMalloc((void **)&states, 8 * (size_t)pool));
  CU(cudaMalloc((void **)&tstar, 8 * (size_t)pool));
  CU(cudaMalloc((void **)&best_s, 4 * (size_t)pool));
  CU(cudaMalloc((void **)&winner, 4));
  CK(hapt_dp_sweep_batch(&t, t.pool, pool, ftop, states, NULL, ws, ws_bytes, NULL));
  CK(hapt_dp_select(ftop, t.pool, pool, t.s_max, B, tstar, best_s, winner, NULL));
  int32_t w, bs;
  double tm, ts;
  CU(cudaMemcpy(&w, winner, 4, cudaMemcpyDeviceToHost));
  if (w < 0) {
    printf("infeasible\n");
    return 0;
  }
  CU(cudaMemcpy(&bs, best_s + w, 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&tm, t.pool + w, 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&ts, tstar + w, 8, cudaMemcpyDeviceToHost));
  /* the winner's stage chain */
  const size_t bt_bytes = hapt_backtrack_workspace_bytes(&t);
  void *bt = NULL;
  int32_t *stages = NULL, *kchain = NULL, *ns = NULL;
  CU(cudaMalloc(&bt, bt_bytes));
  CU(cudaMalloc((void **)&stages, 12 * (size_t)t.s_max));
  CU(cudaMalloc((void **)&kchain, 4 * (size_t)t.s_max));
  CU(cudaMalloc((void **)&ns, 4));
  CK(hapt_dp_backtrack(&t, tm, bs, stages, kchain, ns, bt, bt_bytes, NULL));
  int32_t n;
  CU(cudaMemcpy(&n, ns, 4, cudaMemcpyDeviceToHost));
  int32_t *hs = malloc(12 * (size_t)(n > 0 ? n : 1));
  if (n > 0) CU(cudaMemcpy(hs, stages, 12 * (size_t)n, cudaMemcpyDeviceToHost));
  printf("%.17g %.17g %d %d", tm, ts, bs, n);
  for (int i = 0; i < n; ++i) printf(" %d %d %d", hs[3 * i], hs[3 * i + 1], hs[3 * i + 2]);
  printf("\n");
  return 0;
}
