// Host-side sweep planner (pure C++, no CUDA): turns (n, precision, p) into
// the list of sweeps the engine launches.  See DESIGN.md §3.1.
//
//   groups   G_1 = tile bits [0,K) (contiguous tiles; "A"), then high groups
//            of <= K - m_min target qubits each, tile = 2^m contiguous runs.
//   order    the mixer qubits of one layer commute, so layer k visits the
//            groups forward or backward ("ping-pong"); the last group of
//            layer k is the first of layer k+1 and one sweep does
//            mix_k(X) -> phase_{k+1} -> mix_{k+1}(X).  The last layer ends on
//            G_1 so the final reductions see contiguous tiles (sampler CDF).
//   passes   1 + p*(S-1) HBM round trips for S groups (first one write-only)
//            versus n + p(E_n + n) in the reference's per-gate engine.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

namespace lrq {

struct PlanRound {
  int lo;
  unsigned m1, m2;
  bool phase, reduce;
};

struct PlanGroup {
  int m, q0;          // tile map
  unsigned tmask;     // tile bits that are mixer targets
  std::vector<int> layouts;  // register layouts, first one I/O capable
  int ntargets;
};

struct PlanSweep {
  int group;
  bool init, store;
  int beta1, beta2;   // layer index of mixer 1 / 2 (-1: none)
  int phase;          // layer index of the cost phase (-1: none)
  bool reduce;
  std::vector<PlanRound> rounds;
  int store_lo;
};

struct Plan {
  int n, K, RB, NTB;
  bool small;  // n < K: whole-state kernel
  std::vector<PlanGroup> groups;
  std::vector<PlanSweep> sweeps;
};

inline bool plan_io_ok(const PlanGroup& g, int lo, int RB) {
  if (!(lo >= g.m || lo + RB <= g.m)) return false;  // register bits on one side of m
  return lo >= 3 || g.m <= lo;                        // lanes cover >= 8 contiguous amplitudes
}

inline std::vector<PlanGroup> plan_groups(int n, int K, int RB, int kmax) {
  std::vector<PlanGroup> gs;
  PlanGroup a;
  a.m = K;
  a.q0 = K;
  a.tmask = (K >= 32) ? 0xffffffffu : ((1u << K) - 1u);
  a.ntargets = K;
  // first layout: top register block (I/O capable); then 0, RB, 2RB, ...
  a.layouts.push_back(K - RB);
  for (int lo = 0; lo < K - RB; lo += RB) a.layouts.push_back(lo);
  gs.push_back(a);
  for (int g0 = K; g0 < n; g0 += kmax) {
    const int k = (n - g0) < kmax ? (n - g0) : kmax;
    const int kk = k > RB ? k : RB;
    PlanGroup h;
    h.m = K - kk;
    h.q0 = (k >= RB) ? g0 : g0 + k - RB;
    h.tmask = 0;
    for (int i = h.m; i < K; ++i) {
      const int gp = h.q0 + (i - h.m);
      if (gp >= g0 && gp < g0 + k) h.tmask |= 1u << i;
    }
    h.ntargets = k;
    for (int lo = K - RB; lo > h.m; lo -= RB) h.layouts.push_back(lo);
    if (h.layouts.empty() || h.layouts.back() != h.m) {
      // last layout starts at m (may overlap the previous one)
      bool covered = true;
      unsigned cov = 0;
      for (int lo : h.layouts) cov |= ((1u << RB) - 1u) << lo;
      if ((cov & h.tmask) != h.tmask) covered = false;
      if (!covered) h.layouts.push_back(h.m);
    }
    gs.push_back(h);
  }
  return gs;
}

// greedy assignment of target bits to the rounds of one traversal
inline std::vector<unsigned> plan_masks(const PlanGroup& g, const std::vector<int>& order, int RB) {
  std::vector<unsigned> out;
  unsigned rem = g.tmask;
  for (int lo : order) {
    const unsigned reg = ((1u << RB) - 1u) << lo;
    const unsigned take = rem & reg;
    rem &= ~take;
    out.push_back(take >> lo);
  }
  return out;
}

inline Plan make_plan(int n, int NTB, int RB, int p, int kmax) {
  Plan P;
  P.n = n;
  P.NTB = NTB;
  P.RB = RB;
  P.K = NTB + RB;
  P.small = n < P.K;
  if (P.small || p < 1) return P;
  P.groups = plan_groups(n, P.K, RB, kmax);
  const int S = (int)P.groups.size();

  // op stream: INIT, then per layer PHASE_k, MIX_k(g) for g in the layer order
  struct Op { int kind; int layer; int group; };  // kind 0 phase, 1 mix
  std::vector<Op> ops;
  for (int k = 0; k < p; ++k) {
    ops.push_back({0, k, -1});
    const bool reversed = ((p - 1 - k) % 2) == 0;  // last layer reversed -> ends on G_1
    for (int i = 0; i < S; ++i) ops.push_back({1, k, reversed ? S - 1 - i : i});
  }
  // greedy fusion: [init|load] [mix1 X] [phase] [mix2 X] [reduce if last & X==0]
  size_t i = 0;
  bool first = true;
  while (i < ops.size()) {
    PlanSweep sw;
    sw.init = first;
    sw.store = true;
    sw.beta1 = sw.beta2 = sw.phase = -1;
    sw.reduce = false;
    // group of this sweep: the first mix op at or after i
    size_t j = i;
    while (j < ops.size() && ops[j].kind != 1) ++j;
    sw.group = ops[j].group;
    if (!first && ops[i].kind == 1 && ops[i].group == sw.group) {
      sw.beta1 = ops[i].layer;
      ++i;
    }
    if (i < ops.size() && ops[i].kind == 0) {
      sw.phase = ops[i].layer;
      ++i;
      if (i < ops.size() && ops[i].kind == 1 && ops[i].group == sw.group) {
        sw.beta2 = ops[i].layer;
        ++i;
      }
    }
    if (i == ops.size()) sw.reduce = true;  // planner guarantees group 0 here
    first = false;

    const PlanGroup& g = P.groups[sw.group];
    const std::vector<int>& L = g.layouts;
    std::vector<int> fwd(L.begin(), L.end()), rev(L.rbegin(), L.rend());
    if (sw.beta1 >= 0 && sw.beta2 >= 0) {
      std::vector<unsigned> a = plan_masks(g, fwd, RB), b = plan_masks(g, rev, RB);
      for (size_t r = 0; r < fwd.size(); ++r) sw.rounds.push_back({fwd[r], a[r], 0u, false, false});
      sw.rounds.back().phase = true;
      sw.rounds.back().m2 = b[0];
      for (size_t r = 1; r < rev.size(); ++r) sw.rounds.push_back({rev[r], 0u, b[r], false, false});
    } else if (sw.beta1 >= 0) {
      std::vector<unsigned> a = plan_masks(g, fwd, RB);
      for (size_t r = 0; r < fwd.size(); ++r) sw.rounds.push_back({fwd[r], a[r], 0u, false, false});
    } else {
      // [init|load] phase mix2 : phase in the last layout, mix2 backwards
      std::vector<unsigned> b = plan_masks(g, rev, RB);
      for (size_t r = 0; r < rev.size(); ++r)
        sw.rounds.push_back({rev[r], 0u, sw.beta2 >= 0 ? b[r] : 0u, false, false});
      sw.rounds.front().phase = sw.phase >= 0;
    }
    if (sw.reduce) sw.rounds.back().reduce = true;
    const int last = sw.rounds.back().lo;
    sw.store_lo = plan_io_ok(g, last, RB) ? last : L.front();
    P.sweeps.push_back(sw);
  }
  return P;
}

inline std::string plan_json(const Plan& P) {
  std::string s = "{\"n\":" + std::to_string(P.n) + ",\"K\":" + std::to_string(P.K) +
                  ",\"RB\":" + std::to_string(P.RB) + ",\"small\":" + (P.small ? "true" : "false") +
                  ",\"groups\":[";
  for (size_t i = 0; i < P.groups.size(); ++i) {
    const PlanGroup& g = P.groups[i];
    s += (i ? "," : "");
    s += "{\"m\":" + std::to_string(g.m) + ",\"q0\":" + std::to_string(g.q0) + ",\"tmask\":" +
         std::to_string(g.tmask) + ",\"layouts\":[";
    for (size_t j = 0; j < g.layouts.size(); ++j) s += (j ? "," : "") + std::to_string(g.layouts[j]);
    s += "]}";
  }
  s += "],\"sweeps\":[";
  for (size_t i = 0; i < P.sweeps.size(); ++i) {
    const PlanSweep& w = P.sweeps[i];
    s += (i ? "," : "");
    s += "{\"group\":" + std::to_string(w.group) + ",\"init\":" + (w.init ? "true" : "false") +
         ",\"beta1\":" + std::to_string(w.beta1) + ",\"phase\":" + std::to_string(w.phase) +
         ",\"beta2\":" + std::to_string(w.beta2) + ",\"reduce\":" + (w.reduce ? "true" : "false") +
         ",\"store_lo\":" + std::to_string(w.store_lo) + ",\"rounds\":[";
    for (size_t r = 0; r < w.rounds.size(); ++r) {
      const PlanRound& R = w.rounds[r];
      s += (r ? "," : "");
      s += "[" + std::to_string(R.lo) + "," + std::to_string(R.m1) + "," + std::to_string(R.m2) + "," +
           (R.phase ? "1" : "0") + "," + (R.reduce ? "1" : "0") + "]";
    }
    s += "]}";
  }
  s += "]}";
  return s;
}

}  // namespace lrq
