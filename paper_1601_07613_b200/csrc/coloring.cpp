// Host-side fixed-palette surface coloring, bit-exact with the reference.
//
// Restates the two-stage algorithm of
//   /root/reference/pkg/src/meshchroma/coloring.py
//     _greedy_pass  :138-166   (random free color per surface, -1 if none)
//     _repair       :207-332   (FIFO conflict walk: resolve / swap /
//                               loop-break / forced reswap)
//     color         :395-459   (one RNG stream for greedy+repair, restart
//                               with seed+attempt on budget exhaustion)
//     naive_greedy  :462-488   (first-fit baseline, unbounded palette)
// in C++ so that c4-sized meshes color in seconds instead of minutes.
//
// Bit-exactness hinges on reproducing CPython's `random.Random(seed)`:
// MT19937 seeded through init_by_array() with the 32-bit little-endian
// words of |seed|, and random() = genrand_res53().  A draw happens only when
// more than one choice exists (coloring.py:158, 237, 276-277, 309), choice
// lists are in ascending color order (_MASK_CHOICES, :33-35) and carriers are
// found by scanning the element's surfaces in local side order (:200-204).
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mc_internal.h"

namespace {

// ---------------------------------------------------------------- MT19937
class PyRandom {
 public:
  explicit PyRandom(int64_t seed) {
    uint64_t mag = seed < 0 ? uint64_t(0) - uint64_t(seed) : uint64_t(seed);
    uint32_t key[2];
    int nkey = 0;
    key[nkey++] = uint32_t(mag & 0xffffffffu);
    if (mag >> 32) key[nkey++] = uint32_t(mag >> 32);
    init_by_array(key, nkey);
  }

  // genrand_res53: 53-bit double in [0, 1)
  double random() {
    uint32_t a = next() >> 5, b = next() >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
  }

  // CPython's int(random() * n)
  int pick(int n) { return int(random() * double(n)); }

 private:
  static constexpr int N = 624, M = 397;
  uint32_t mt_[N];
  int mti_ = N + 1;

  void init_genrand(uint32_t s) {
    mt_[0] = s;
    for (mti_ = 1; mti_ < N; ++mti_)
      mt_[mti_] = 1812433253u * (mt_[mti_ - 1] ^ (mt_[mti_ - 1] >> 30)) + uint32_t(mti_);
  }

  void init_by_array(const uint32_t* key, int len) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = (N > len ? N : len); k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1664525u)) + key[j] + uint32_t(j);
      ++i;
      ++j;
      if (i >= N) { mt_[0] = mt_[N - 1]; i = 1; }
      if (j >= len) j = 0;
    }
    for (int k = N - 1; k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1566083941u)) - uint32_t(i);
      ++i;
      if (i >= N) { mt_[0] = mt_[N - 1]; i = 1; }
    }
    mt_[0] = 0x80000000u;
  }

  uint32_t next() {
    if (mti_ >= N) {
      int kk = 0;
      uint32_t y;
      for (; kk < N - M; ++kk) {
        y = (mt_[kk] & 0x80000000u) | (mt_[kk + 1] & 0x7fffffffu);
        mt_[kk] = mt_[kk + M] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      for (; kk < N - 1; ++kk) {
        y = (mt_[kk] & 0x80000000u) | (mt_[kk + 1] & 0x7fffffffu);
        mt_[kk] = mt_[kk + (M - N)] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      }
      y = (mt_[N - 1] & 0x80000000u) | (mt_[0] & 0x7fffffffu);
      mt_[N - 1] = mt_[M - 1] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
      mti_ = 0;
    }
    uint32_t y = mt_[mti_++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
  }
};

// colors (1..7) present in a bitmask, ascending
inline int mask_colors(uint32_t m, int* out) {
  int n = 0;
  for (int c = 1; c < 8; ++c)
    if ((m >> c) & 1u) out[n++] = c;
  return n;
}

struct Incidence {
  int64_t ns = 0, ne = 0;
  std::vector<int32_t> left, right;
  std::vector<int32_t> es;      // element surfaces, -1 entries dropped, 4 slots
  std::vector<uint8_t> es_n;    // surfaces per element
};

bool load_incidence(int64_t ns, int64_t ne, const int64_t* surf_elems,
                    const int64_t* elem_surfs, Incidence& inc) {
  if (ns < 0 || ne < 0 || ns >= (int64_t(1) << 31) || ne >= (int64_t(1) << 31)) {
    mc_set_error("mesh too large for 32-bit incidence");
    return false;
  }
  inc.ns = ns;
  inc.ne = ne;
  inc.left.resize(ns);
  inc.right.resize(ns);
  for (int64_t k = 0; k < ns; ++k) {
    int64_t l = surf_elems[2 * k], r = surf_elems[2 * k + 1];
    if (l < 0 || l >= ne || r >= ne) {
      mc_set_error("surface " + std::to_string(k) + " has an out-of-range element");
      return false;
    }
    inc.left[k] = int32_t(l);
    inc.right[k] = r >= 0 ? int32_t(r) : -1;
  }
  if (elem_surfs) {
    inc.es.assign(size_t(ne) * 4, -1);
    inc.es_n.assign(ne, 0);
    for (int64_t e = 0; e < ne; ++e) {
      int n = 0;
      for (int j = 0; j < 4; ++j) {
        int64_t s = elem_surfs[4 * e + j];
        if (s >= 0) inc.es[4 * e + n++] = int32_t(s);
      }
      inc.es_n[e] = uint8_t(n);
    }
  }
  return true;
}

struct RepairStats {
  int64_t resolutions = 0, swaps = 0, loop_breaks = 0, no_swap_breaks = 0,
          forced_reswaps = 0;
};

enum class RepairOutcome { kDone, kBudget, kInternal, kAudit };

class Colorer {
 public:
  Colorer(const Incidence& inc, int n_colors)
      : inc_(inc), n_colors_(n_colors),
        full_(((1u << n_colors) - 1u) << 1) {}

  // coloring.py:138-166
  void greedy(PyRandom& rng, std::vector<int32_t>& colors,
              std::vector<uint32_t>& used, std::vector<int32_t>& conflicts) {
    const int64_t ns = inc_.ns;
    colors.assign(ns, -1);
    used.assign(inc_.ne, 0u);
    conflicts.clear();
    int t[8];
    for (int64_t k = 0; k < ns; ++k) {
      int32_t l = inc_.left[k], r = inc_.right[k];
      uint32_t ul = used[l], ur = r >= 0 ? used[r] : 0u;
      uint32_t m = full_ & ~(ul | ur);
      if (m) {
        int n = mask_colors(m, t);
        int c = n == 1 ? t[0] : t[rng.pick(n)];
        colors[k] = c;
        uint32_t b = 1u << c;
        used[l] = ul | b;
        if (r >= 0) used[r] = ur | b;
      } else {
        conflicts.push_back(int32_t(k));
      }
    }
  }

  // coloring.py:207-332
  RepairOutcome repair(PyRandom& rng, std::vector<int32_t>& colors,
                       std::vector<uint32_t>& used,
                       const std::vector<int32_t>& conflicts,
                       int64_t chain_budget, int64_t total_budget, bool audit,
                       RepairStats& st, std::string& msg) {
    std::vector<int32_t> queue(conflicts.begin(), conflicts.end());
    size_t head = 0;
    std::vector<uint32_t> stamp(inc_.ns, 0u);
    uint32_t chain_id = 0;
    int64_t total_swaps = 0;
    struct Move { int c; int32_t a, b; };
    Move cand[8], stale[8], brk[8];
    int t[8];

    while (head < queue.size()) {
      int32_t e = queue[head++];
      if (colors[e] != -1) continue;
      ++chain_id;
      stamp[e] = chain_id;
      int64_t chain_swaps = 0;
      for (;;) {
        const int32_t l = inc_.left[e], r = inc_.right[e];
        const uint32_t ul = used[l], ur = r >= 0 ? used[r] : 0u;
        const uint32_t m = full_ & ~(ul | ur);
        if (m) {
          int n = mask_colors(m, t);
          int c = n == 1 ? t[0] : t[rng.pick(n)];
          colors[e] = c;
          uint32_t b = 1u << c;
          used[l] = ul | b;
          if (r >= 0) used[r] = ur | b;
          ++st.resolutions;
          if (audit && !check(colors, msg)) return RepairOutcome::kAudit;
          break;
        }
        const uint32_t both = ul & ur;
        const uint32_t single = (ul | ur) ^ both;
        int nc = 0, nst = 0, nb = 0;
        if (single) {
          int n = mask_colors(single, t);
          for (int q = 0; q < n; ++q) {
            int c = t[q];
            int32_t owner = ((ul >> c) & 1u) ? l : r;
            int32_t s = carrier(owner, colors, c);
            if (s < 0) { msg = "no surface of color " + std::to_string(c) + " on element"; return RepairOutcome::kInternal; }
            if (stamp[s] == chain_id) stale[nst++] = {c, s, -1};
            else cand[nc++] = {c, s, -1};
          }
        }
        if (both) {
          int n = mask_colors(both, t);
          for (int q = 0; q < n; ++q) {
            int c = t[q];
            int32_t ea = carrier(l, colors, c), eb = carrier(r, colors, c);
            if (ea < 0 || eb < 0) { msg = "no surface of color " + std::to_string(c) + " on element"; return RepairOutcome::kInternal; }
            if (ea == eb) {
              if (stamp[ea] == chain_id) stale[nst++] = {c, ea, -1};
              else cand[nc++] = {c, ea, -1};
            } else {
              brk[nb++] = {c, ea, eb};
            }
          }
        }
        const Move* pool = cand;
        int npool = nc;
        if (nc == 0) {
          if (nb) {
            const Move& mv = nb == 1 ? brk[0] : brk[rng.pick(nb)];
            uint32_t b = 1u << mv.c;
            for (int32_t s : {mv.a, mv.b}) {
              colors[s] = -1;
              used[inc_.left[s]] &= ~b;
              int32_t rs = inc_.right[s];
              if (rs >= 0) used[rs] &= ~b;
            }
            colors[e] = mv.c;
            used[l] |= b;
            if (r >= 0) used[r] |= b;
            queue.push_back(mv.a);
            queue.push_back(mv.b);
            if (nst || single) ++st.loop_breaks;
            else ++st.no_swap_breaks;
            if (audit && !check(colors, msg)) return RepairOutcome::kAudit;
            break;
          }
          if (nst == 0) {
            msg = "conflict on surface " + std::to_string(e) + " has no admissible move";
            return RepairOutcome::kBudget;
          }
          pool = stale;
          npool = nst;
          ++st.forced_reswaps;
        }
        const Move& mv = npool == 1 ? pool[0] : pool[rng.pick(npool)];
        const int32_t es = mv.a;
        const uint32_t b = 1u << mv.c;
        colors[es] = -1;
        used[inc_.left[es]] &= ~b;
        int32_t rs = inc_.right[es];
        if (rs >= 0) used[rs] &= ~b;
        colors[e] = mv.c;
        used[l] |= b;
        if (r >= 0) used[r] |= b;
        ++st.swaps;
        ++chain_swaps;
        ++total_swaps;
        if (audit && !check(colors, msg)) return RepairOutcome::kAudit;
        if (chain_swaps > chain_budget || total_swaps > total_budget) {
          msg = "spent " + std::to_string(chain_swaps) +
                " swaps on one conflict chain (" + std::to_string(total_swaps) +
                " in total)";
          return RepairOutcome::kBudget;
        }
        stamp[es] = chain_id;
        e = es;
      }
    }
    return RepairOutcome::kDone;
  }

 private:
  const Incidence& inc_;
  int n_colors_;
  uint32_t full_;

  int32_t carrier(int32_t elem, const std::vector<int32_t>& colors, int c) const {
    const int32_t* row = &inc_.es[size_t(elem) * 4];
    for (int j = 0; j < inc_.es_n[elem]; ++j)
      if (colors[row[j]] == c) return row[j];
    return -1;
  }

  // audit (coloring.py:335-348): no element sees a color twice
  bool check(const std::vector<int32_t>& colors, std::string& msg) const {
    std::vector<uint32_t> seen(inc_.ne, 0u);
    for (int64_t k = 0; k < inc_.ns; ++k) {
      int c = colors[k];
      if (c < 1) continue;
      uint32_t b = 1u << c;
      for (int32_t e : {inc_.left[k], inc_.right[k]}) {
        if (e < 0) continue;
        if (seen[e] & b) {
          msg = "color " + std::to_string(c) + " repeated on element " + std::to_string(e);
          return false;
        }
        seen[e] |= b;
      }
    }
    return true;
  }
};

double now_s() {
  using clk = std::chrono::steady_clock;
  return std::chrono::duration<double>(clk::now().time_since_epoch()).count();
}

void copy_stats(const RepairStats& st, mc_coloring_stats* out) {
  if (!out) return;
  out->resolutions = st.resolutions;
  out->swaps = st.swaps;
  out->loop_breaks = st.loop_breaks;
  out->no_swap_breaks = st.no_swap_breaks;
  out->forced_reswaps = st.forced_reswaps;
}

}  // namespace

extern "C" {

MC_API int mc_color(int64_t n_surfaces, int64_t n_elements,
                    const int64_t* surf_elems, const int64_t* elem_surfs,
                    int n_colors, int64_t seed, int64_t chain_budget,
                    int max_restarts, int audit, int32_t* colors_out,
                    mc_coloring_stats* stats) {
  if (n_surfaces <= 0) return mc_fail(MC_EINVAL, "mesh has no surfaces");
  if (n_colors < 1 || n_colors > 7) return mc_fail(MC_EINVAL, "palette must have 1..7 colors");
  Incidence inc;
  if (!load_incidence(n_surfaces, n_elements, surf_elems, elem_surfs, inc)) return MC_EINVAL;
  if (chain_budget < 0) chain_budget = 10 * n_surfaces;
  Colorer col(inc, n_colors);
  std::vector<int32_t> colors, conflicts;
  std::vector<uint32_t> used;
  std::string last;
  const double t_start = now_s();
  for (int attempt = 0; attempt <= max_restarts; ++attempt) {
    PyRandom rng(seed + attempt);
    const double t0 = now_s();
    col.greedy(rng, colors, used, conflicts);
    const double t1 = now_s();
    RepairStats st;
    std::string msg;
    RepairOutcome out = col.repair(rng, colors, used, conflicts, chain_budget,
                                   5 * chain_budget, audit != 0, st, msg);
    if (out == RepairOutcome::kBudget) { last = msg; continue; }
    if (out == RepairOutcome::kAudit) return mc_fail(MC_EAUDIT, msg);
    if (out == RepairOutcome::kInternal) return mc_fail(MC_EINTERNAL, msg);
    const double t2 = now_s();
    std::memcpy(colors_out, colors.data(), sizeof(int32_t) * n_surfaces);
    if (stats) {
      copy_stats(st, stats);
      stats->greedy_conflicts = int64_t(conflicts.size());
      stats->restarts = attempt;
      stats->greedy_seconds = t1 - t0;
      stats->resolve_seconds = t2 - t1;
      stats->total_seconds = t2 - t_start;
    }
    return MC_OK;
  }
  return mc_fail(MC_ERESTARTS, "no complete coloring after " +
                                   std::to_string(max_restarts + 1) +
                                   " attempts (last: " + last + ")");
}

MC_API int mc_modified_greedy(int64_t n_surfaces, int64_t n_elements,
                              const int64_t* surf_elems, int n_colors,
                              int64_t seed, int32_t* colors_out,
                              int64_t* n_conflicts) {
  if (n_surfaces <= 0) return mc_fail(MC_EINVAL, "mesh has no surfaces");
  if (n_colors < 1 || n_colors > 7) return mc_fail(MC_EINVAL, "palette must have 1..7 colors");
  Incidence inc;
  if (!load_incidence(n_surfaces, n_elements, surf_elems, nullptr, inc)) return MC_EINVAL;
  Colorer col(inc, n_colors);
  std::vector<int32_t> colors, conflicts;
  std::vector<uint32_t> used;
  PyRandom rng(seed);
  col.greedy(rng, colors, used, conflicts);
  std::memcpy(colors_out, colors.data(), sizeof(int32_t) * n_surfaces);
  if (n_conflicts) *n_conflicts = int64_t(conflicts.size());
  return MC_OK;
}

MC_API int mc_resolve_conflicts(int64_t n_surfaces, int64_t n_elements,
                                const int64_t* surf_elems,
                                const int64_t* elem_surfs, int n_colors,
                                int64_t seed, int64_t chain_budget, int audit,
                                int32_t* colors_inout,
                                mc_coloring_stats* stats) {
  if (n_colors < 1 || n_colors > 7) return mc_fail(MC_EINVAL, "palette must have 1..7 colors");
  Incidence inc;
  if (!load_incidence(n_surfaces, n_elements, surf_elems, elem_surfs, inc)) return MC_EINVAL;
  if (chain_budget < 0) chain_budget = 10 * n_surfaces;
  std::vector<int32_t> colors(colors_inout, colors_inout + n_surfaces);
  std::vector<uint32_t> used(n_elements, 0u);
  std::vector<int32_t> conflicts;
  // coloring.py:169-188: rebuild per-element masks, reject repeats
  for (int64_t k = 0; k < n_surfaces; ++k) {
    int c = colors[k];
    if (c < 1) { conflicts.push_back(int32_t(k)); continue; }
    uint32_t b = 1u << c;
    for (int32_t e : {inc.left[k], inc.right[k]}) {
      if (e < 0) continue;
      if (used[e] & b)
        return mc_fail(MC_EINVAL, "input coloring repeats color " + std::to_string(c) +
                                      " on element " + std::to_string(e));
      used[e] |= b;
    }
  }
  Colorer col(inc, n_colors);
  PyRandom rng(seed);
  RepairStats st;
  std::string msg;
  RepairOutcome out = col.repair(rng, colors, used, conflicts, chain_budget,
                                 5 * chain_budget, audit != 0, st, msg);
  if (out == RepairOutcome::kBudget) return mc_fail(MC_ESWAPBUDGET, msg);
  if (out == RepairOutcome::kAudit) return mc_fail(MC_EAUDIT, msg);
  if (out == RepairOutcome::kInternal) return mc_fail(MC_EINTERNAL, msg);
  std::memcpy(colors_inout, colors.data(), sizeof(int32_t) * n_surfaces);
  if (stats) {
    copy_stats(st, stats);
    stats->greedy_conflicts = int64_t(conflicts.size());
    stats->restarts = 0;
  }
  return MC_OK;
}

MC_API int mc_naive_greedy(int64_t n_surfaces, int64_t n_elements,
                           const int64_t* surf_elems, int32_t* colors_out,
                           int32_t* n_colors_out) {
  if (n_surfaces <= 0) return mc_fail(MC_EINVAL, "mesh has no surfaces");
  Incidence inc;
  if (!load_incidence(n_surfaces, n_elements, surf_elems, nullptr, inc)) return MC_EINVAL;
  std::vector<uint64_t> used(n_elements, 0u);
  int top = 0;
  for (int64_t k = 0; k < n_surfaces; ++k) {
    int32_t l = inc.left[k], r = inc.right[k];
    uint64_t m = used[l] | (r >= 0 ? used[r] : 0u);
    int c = 1;
    while ((m >> c) & 1u) ++c;
    colors_out[k] = c;
    if (c > top) top = c;
    used[l] |= uint64_t(1) << c;
    if (r >= 0) used[r] |= uint64_t(1) << c;
  }
  if (n_colors_out) *n_colors_out = top;
  return MC_OK;
}

}  // extern "C"
