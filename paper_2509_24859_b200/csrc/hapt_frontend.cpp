// Model-graph front end: repeated-module detection and
// min-max layer clustering, native host code.
//
// Reference: meshpipe.model_graph (model_graph.py:112-333), pure Python and
// O(n * max_len) tuple-hashing per detection round -- 16-26 s at the 2,006-op
// config D graph, longer than the whole GPU search it feeds.
//
//  * detect_modules: per pattern length, every admissible window (>= z heavy
//    ops) is keyed by a 64-bit polynomial hash of its tag ids; windows are
//    grouped by hash AND verified equal element-wise against the group's
//    first window, so grouping is exactly the reference's dict of tag
//    tuples.  Greedy non-overlapping counts and the (count, length,
//    -first position) max are the reference's (model_graph.py:112-166);
//    the scan stops at the first repeat-free length when z == 1, like the
//    reference, and as soon as sum(span // length) -- an upper bound on any
//    longer window's count -- drops below the best count found (config D:
//    ~64 lengths scanned instead of ~1,000; same result).
//  * cluster_layers: the min-max contiguous partition DP of
//    model_graph.py:235-266 in the same fp64 expression order (earliest
//    cuts on ties); layer flops / param bytes are CPython sums, which are
//    compensated on Python >= 3.12 (Neumaier), so they are reproduced with
//    the same algorithm to stay bit-identical.
//
// All pointers are HOST memory; no CUDA involvement.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <unordered_map>
#include <vector>

#include "../../include/hapt_b200.h"

namespace hapt {
void set_error(const char *fmt, ...);
}

namespace {

struct Found {
  int count = 0, length = 0, first = 0;
  std::vector<int> chosen;
};

// _best_pattern (model_graph.py:123-166)
bool best_pattern(const std::vector<int> &tags, const std::vector<int> &heavy_prefix,
                  const std::vector<std::pair<int, int>> &spans, int z, Found &best) {
  const int n = (int)tags.size();
  int max_len = 0;
  for (auto &sp : spans) max_len = std::max(max_len, sp.second - sp.first);
  // prefix polynomial hashes (mod 2^64)
  const uint64_t base = 0x9E3779B97F4A7C15ull;
  std::vector<uint64_t> P(n + 1, 0), pw(n + 1, 1);
  for (int i = 0; i < n; ++i) {
    P[i + 1] = P[i] * base + (uint64_t)(uint32_t)tags[i] + 1;
    pw[i + 1] = pw[i] * base;
  }
  bool have = false;
  struct Group {
    int first;               // first window (pattern representative)
    std::vector<int> pos;    // ascending
  };
  std::unordered_map<uint64_t, std::vector<int>> by_hash;  // hash -> group ids
  std::vector<Group> groups;
  for (int length = 1; length <= max_len; ++length) {
    long fit = 0;
    for (auto &sp : spans) fit += (sp.second - sp.first) / length;
    if (fit < 2) break;
    // no window of this length or longer can repeat more often than `fit`
    // (non-increasing in length), and the key is count first: once that
    // bound falls below the best count found, no later length can win
    if (have && fit < best.count) break;
    by_hash.clear();
    groups.clear();
    for (auto &sp : spans) {
      for (int pos = sp.first; pos + length <= sp.second; ++pos) {
        if (heavy_prefix[pos + length] - heavy_prefix[pos] < z) continue;
        const uint64_t h = P[pos + length] - P[pos] * pw[length];
        auto &ids = by_hash[h];
        int gid = -1;
        for (int cand : ids) {
          const int f = groups[cand].first;
          if (memcmp(&tags[f], &tags[pos], sizeof(int) * length) == 0) {
            gid = cand;
            break;
          }
        }
        if (gid < 0) {
          gid = (int)groups.size();
          groups.push_back(Group{pos, {}});
          ids.push_back(gid);
        }
        groups[gid].pos.push_back(pos);
      }
    }
    bool repeated_here = false;
    for (auto &gr : groups) {
      // _greedy_positions: left-to-right non-overlapping selection
      int cnt = 0, last_end = -1, first = -1;
      for (int p : gr.pos)
        if (p >= last_end) {
          if (cnt == 0) first = p;
          ++cnt;
          last_end = p + length;
        }
      if (cnt < 2) continue;
      repeated_here = true;
      // key (count, length, -first) maximised
      const bool better = !have || cnt > best.count ||
                          (cnt == best.count && (length > best.length ||
                                                 (length == best.length && first < best.first)));
      if (better) {
        have = true;
        best.count = cnt;
        best.length = length;
        best.first = first;
        best.chosen.clear();
        last_end = -1;
        for (int p : gr.pos)
          if (p >= last_end) {
            best.chosen.push_back(p);
            last_end = p + length;
          }
      }
    }
    // for z = 1 a repeating pattern of length L+1 embeds a repeating window
    // of length L, so the first repeat-free length ends the scan
    if (!repeated_here && z == 1) break;
  }
  return have;
}

// CPython >= 3.12 builtin sum() over floats: int start 0, then Neumaier
// compensated summation (bltinmodule.c builtin_sum_impl).
double py_sum(const double *x, int n) {
  if (n <= 0) return 0.0;
  double f = 0.0 + x[0];
  double c = 0.0;
  for (int i = 1; i < n; ++i) {
    const double xi = x[i];
    const double t = f + xi;
    if (fabs(f) >= fabs(xi))
      c += (f - t) + xi;
    else
      c += (xi - t) + f;
    f = t;
  }
  if (c != 0.0 && isfinite(c)) f += c;
  return f;
}

// _min_max_partition (model_graph.py:235-266): cut positions (exclusive ends)
std::vector<int> min_max_partition(const double *values, int n, int parts) {
  std::vector<double> prefix(n + 1, 0.0);
  for (int i = 0; i < n; ++i) prefix[i + 1] = prefix[i] + values[i];
  const double INF = HUGE_VAL;
  std::vector<std::vector<double>> best(parts + 1, std::vector<double>(n + 1, INF));
  std::vector<std::vector<int>> cut(parts + 1, std::vector<int>(n + 1, -1));
  best[0][0] = 0.0;
  for (int p = 1; p <= parts; ++p) {
    for (int j = p; j <= n - (parts - p); ++j) {
      for (int i = p - 1; i < j; ++i) {
        if (best[p - 1][i] == INF) continue;
        const double cand = std::max(best[p - 1][i], prefix[j] - prefix[i]);
        if (cand < best[p][j]) {
          best[p][j] = cand;
          cut[p][j] = i;
        }
      }
    }
  }
  std::vector<int> cuts;
  int j = n;
  for (int p = parts; p >= 1; --p) {
    cuts.push_back(j);
    j = cut[p][j];
  }
  std::reverse(cuts.begin(), cuts.end());
  return cuts;
}

}  // namespace

extern "C" int hapt_detect_modules(int32_t n_ops, const int32_t *tag_host,
                                   const uint8_t *heavy_host, int32_t z, int32_t *span_start,
                                   int32_t *span_end, int32_t *span_group, int32_t *span_occ,
                                   int32_t *n_spans) {
  if (n_ops < 1 || !tag_host || !heavy_host || z < 1 || !span_start || !span_end ||
      !span_group || !span_occ || !n_spans) {
    hapt::set_error("hapt_detect_modules: invalid arguments");
    return HAPT_EINVAL;
  }
  std::vector<int> tags(tag_host, tag_host + n_ops);
  std::vector<int> heavy_prefix(n_ops + 1, 0);
  for (int i = 0; i < n_ops; ++i) heavy_prefix[i + 1] = heavy_prefix[i] + (heavy_host[i] ? 1 : 0);
  struct Span {
    int start, end, group, occ;
  };
  std::vector<Span> repeated;
  std::vector<std::pair<int, int>> free_spans{{0, n_ops}};
  int group_id = 0;
  Found f;
  while (best_pattern(tags, heavy_prefix, free_spans, z, f)) {
    for (size_t occ = 0; occ < f.chosen.size(); ++occ)
      repeated.push_back({f.chosen[occ], f.chosen[occ] + f.length, group_id, (int)occ});
    ++group_id;
    std::vector<std::pair<int, int>> occupied;
    for (auto &s : repeated) occupied.push_back({s.start, s.end});
    std::sort(occupied.begin(), occupied.end());
    free_spans.clear();
    int cursor = 0;
    for (auto &o : occupied) {
      if (cursor < o.first) free_spans.push_back({cursor, o.first});
      cursor = o.second;
    }
    if (cursor < n_ops) free_spans.push_back({cursor, n_ops});
    f = Found();
  }
  std::vector<Span> all = repeated;
  for (auto &fs : free_spans) all.push_back({fs.first, fs.second, -1, 0});
  std::stable_sort(all.begin(), all.end(),
                   [](const Span &a, const Span &b) { return a.start < b.start; });
  for (size_t i = 0; i < all.size(); ++i) {
    span_start[i] = all[i].start;
    span_end[i] = all[i].end;
    span_group[i] = all[i].group;
    span_occ[i] = all[i].occ;
  }
  *n_spans = (int32_t)all.size();
  return HAPT_OK;
}

extern "C" int hapt_cluster_layers(int32_t n_ops, const double *flops_host,
                                   const double *params_host, const double *out_bytes_host,
                                   int32_t n_spans, const int32_t *span_start,
                                   const int32_t *span_end, const int32_t *span_group,
                                   int32_t u, int32_t *layer_start, int32_t *layer_end,
                                   double *layer_flops, double *layer_params,
                                   double *layer_bbytes, int32_t *layer_sig,
                                   int32_t *n_layers) {
  if (n_ops < 1 || n_spans < 1 || u < 1 || !flops_host || !params_host || !out_bytes_host ||
      !span_start || !span_end || !span_group || !layer_start || !layer_end || !layer_flops ||
      !layer_params || !layer_bbytes || !layer_sig || !n_layers) {
    hapt::set_error("hapt_cluster_layers: invalid arguments");
    return HAPT_EINVAL;
  }
  std::unordered_map<int, std::vector<int>> group_cuts;
  int n = 0, solo = 0;
  for (int sp = 0; sp < n_spans; ++sp) {
    const int s0 = span_start[sp], s1 = span_end[sp], grp = span_group[sp];
    if (u > s1 - s0) {
      hapt::set_error("span %d has %d operators, cannot form %d layers", sp, s1 - s0, u);
      return HAPT_EINVAL;
    }
    std::vector<int> cuts;
    if (grp >= 0) {
      auto it = group_cuts.find(grp);
      if (it == group_cuts.end())
        it = group_cuts.emplace(grp, min_max_partition(flops_host + s0, s1 - s0, u)).first;
      cuts = it->second;
    } else {
      cuts = min_max_partition(flops_host + s0, s1 - s0, u);
    }
    int prev = 0;
    for (int part = 0; part < (int)cuts.size(); ++part) {
      const int lo = s0 + prev, hi = s0 + cuts[part];
      layer_start[n] = lo;
      layer_end[n] = hi;
      layer_flops[n] = py_sum(flops_host + lo, hi - lo);
      layer_params[n] = py_sum(params_host + lo, hi - lo);
      layer_bbytes[n] = out_bytes_host[hi - 1];
      layer_sig[3 * n + 0] = grp >= 0 ? 0 : 1;  // "rep" / "solo"
      layer_sig[3 * n + 1] = grp >= 0 ? grp : solo;
      layer_sig[3 * n + 2] = part;
      ++n;
      prev = cuts[part];
    }
    if (grp < 0) ++solo;
  }
  *n_layers = n;
  return HAPT_OK;
}

extern "C" double hapt_py_sum(const double *x_host, int32_t n) { return py_sum(x_host, n); }
