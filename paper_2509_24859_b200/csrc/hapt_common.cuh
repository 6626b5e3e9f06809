// Shared helpers for the HAPT B200 kernels (sm_100a).
//
// Every floating-point expression that the reference evaluates in Python /
// Cython is written with explicit round-to-nearest intrinsics (__dadd_rn,
// __dmul_rn, __ddiv_rn) so that nvcc can never contract it into an FMA; the
// library is additionally compiled with --fmad=false.  This is what makes the
// device tables and DP values bit-identical to the CPU reference
// (SURVEY.md Appendix A).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/hapt_b200.h"

namespace hapt {

constexpr double kInf = __builtin_huge_val();
constexpr int kKSat = 65535;  // saturation of the integer memory threshold

void set_error(const char *fmt, ...);
void note_launch();  // one kernel enqueued by the library (hapt_launches)
void *tables_hist(const hapt_tables *t);  // rank-histogram scratch of a tables buffer

inline int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return HAPT_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return HAPT_ECUDA;
}

#define HAPT_CUDA(call)                                           \
  do {                                                            \
    int _st = ::hapt::cuda_status((call), #call);                 \
    if (_st != HAPT_OK) return _st;                               \
  } while (0)

#define HAPT_LAUNCHED(what)                                       \
  do {                                                            \
    int _st = ::hapt::cuda_status(cudaGetLastError(), what);      \
    if (_st != HAPT_OK) return _st;                               \
  } while (0)

// Programmatic dependent launch (sm_90+).  A kernel enqueued with
// launch_pdl() may be scheduled while its predecessor in the stream drains:
// it calls pdl_wait() before touching anything earlier work wrote (a no-op
// when it was launched normally), then pdl_trigger() so its own successor
// can be scheduled as soon as every block of this grid is resident.  This
// hides the launch gap of the layer-by-layer kernel chain.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

bool pdl_enabled();  // HAPT_PDL=0 disables (A/B measurements)

// Kernel timing (hapt_prof_enable / hapt_prof_read): kinds of timed launches
enum ProfKind { kProfRelax = 0, kProfWindow = 1, kProfOther = 2, kProfKinds = 3 };
bool prof_on();
void *prof_begin(int kind, cudaStream_t st);
void prof_end(void *h, cudaStream_t st);
struct ProfScope {
  void *h;
  cudaStream_t st;
  ProfScope(int kind, cudaStream_t s) : h(prof_begin(kind, s)), st(s) {}
  ~ProfScope() { prof_end(h, st); }
};

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, bool on,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

inline unsigned grid_for(size_t n, unsigned block) {
  size_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (unsigned)g;
}

// Exact memory mask of _dp.pyx:83 turned into an integer threshold: the
// largest integer K in [0, kKSat] with  !(mp + K*ma > cap)  for every
// integer in [1, K].  fl(mp + fl(K*ma)) is monotone non-decreasing in K for
// ma >= 0 (round-to-nearest is monotone), so the admissible K form a prefix
// and  kk <= kmax  is bit-equivalent to the reference test.
__device__ __forceinline__ bool mem_ok(double mp, double ma, double cap, int K) {
  return !(__dadd_rn(mp, __dmul_rn((double)K, ma)) > cap);
}

__device__ __forceinline__ int mem_kmax(double mp, double ma, double cap) {
  if (!mem_ok(mp, ma, cap, 1)) return 0;
  if (mem_ok(mp, ma, cap, kKSat)) return kKSat;
  int lo = 1, hi = kKSat;  // ok(lo), !ok(hi)
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (mem_ok(mp, ma, cap, mid)) lo = mid; else hi = mid;
  }
  return lo;
}

// Positive IEEE doubles order like their bit patterns.
__device__ __forceinline__ unsigned long long dkey(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

}  // namespace hapt
