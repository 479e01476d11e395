// Host-side sweep planner: turns (n, precision, p) into the list of sweeps the
// engine launches.  See DESIGN.md §3.1.
//
//   groups   G_1 = "A" = tile amp bits [0, KA) (one contiguous run per tile),
//            then high groups "H" of <= KA - MA target qubits each; an H tile
//            is 2^(KA-MA) runs of 2^MA contiguous amplitudes.
//   order    the mixer qubits of one layer commute, so layer k visits the
//            groups forward or backward ("ping-pong"); the last group of
//            layer k is the first of layer k+1 and one sweep does
//            mix_k(X) -> phase_{k+1} -> mix_{k+1}(X).  The last layer ends on
//            G_1 so the final reductions see contiguous tiles (sampler CDF).
//   passes   1 + p*(S-1) HBM round trips for S >= 2 groups (the first one is
//            write-only) versus n + p(E_n + n) in the reference's per-gate engine.
//   rounds   the register layouts of each sweep are fixed at compile time per
//            (group kind, sweep kind) (lrq_sweep.cuh prog_*); the planner only
//            assigns which register bits take a butterfly in which round.
#pragma once
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "lrq_sweep.cuh"

namespace lrq {

struct PlanGroup {
  int kind;        // GK_A / GK_H / GK_H4 / GK_C*
  int m, q0;       // tile amp bit i -> global i < m ? i : q0 + (i - m)
  unsigned tmask;  // tile amp bits that are mixer targets
  int ntargets;    // mixer targets of the group (a cluster group: + the cross qubit)
  int cross = -1;  // cluster groups: the target qubit between the two CTAs' half tiles
};

struct PlanSweep {
  int group;
  int kind;                 // SK_*
  int beta1, phase, beta2;  // layer indices (-1: none)
  bool reduce;
  int nrounds;
  unsigned mask1[kMaxRounds], mask2[kMaxRounds];  // register-amp-bit masks
  unsigned tmask1[kMaxRounds], tmask2[kMaxRounds];  // same, as tile amp bits
  // distributed plans: the mixer-1 targets of a sweep can be a subset of the
  // group (the qubits a remap just made local); 0 = the whole group
  unsigned target1;
  int ntarget1, ntarget2;  // qubits mixed by mixer 1 / 2 (scale factor powers)
  bool remap_after;        // distributed plans: a qubit remap follows this sweep
  int perm;                // permutation state the sweep runs in (0 identity, 1 swapped)
  int prog;                // 0: round programs of sweep_kernel / sweep_tma_kernel;
                           // 1: warp-decoupled 2-layout program (lrq_sweep_wd.cuh)
};

struct Plan {
  int n, KA, pair;
  bool small;  // n < KA: whole-state kernel
  std::vector<PlanGroup> groups;
  std::vector<PlanSweep> sweeps;
};

inline std::vector<PlanGroup> plan_groups_tiles(int n, int pair);
inline std::vector<PlanGroup> plan_groups(int n, int pair) { return plan_groups_tiles(n, pair); }
inline std::vector<PlanGroup> plan_groups_tiles(int n, int pair) {
  const int KA = kUnitBits + pair;
  std::vector<PlanGroup> gs;
  PlanGroup a;
  a.kind = GK_A;
  a.m = KA;
  a.q0 = KA;
  a.tmask = (1u << KA) - 1u;
  a.ntargets = KA;
  gs.push_back(a);
  // high groups: as few as possible; for complex64 as many of them as the
  // count allows use 128 B runs (H4, 9 targets), the rest 64 B runs (H, 10)
  const int rest = n > KA ? n - KA : 0;
  const int kH = KA - group_ma(GK_H, pair);
  const int nh = (rest + kH - 1) / kH;
  int n_h4 = 0;
  if (pair) {
    const int kH4 = KA - group_ma(GK_H4, pair);
    const int need10 = rest - kH4 * nh;  // groups that must take 10 targets
    n_h4 = nh - (need10 > 0 ? need10 : 0);
  }
  for (int i = 0, g0 = KA; g0 < n; ++i) {
    // H4 groups last: the top qubits give a group's runs the largest stride
    // (2^q0 amplitudes); 128 B runs tolerate that, 64 B runs do not (n=32:
    // an F sweep on H at q0=22 takes 30 ms, at q0=13 14 ms)
    const int kind = i >= nh - n_h4 ? GK_H4 : GK_H;
    const int MA = group_ma(kind, pair);
    const int kmax = KA - MA;
    const int k = (n - g0) < kmax ? (n - g0) : kmax;
    PlanGroup h;
    h.kind = kind;
    h.m = MA;
    h.q0 = g0 + k - kmax;  // short last group: slide the run down (extra bits are non-targets)
    h.tmask = 0;
    for (int i = MA; i < KA; ++i) {
      const int gp = h.q0 + (i - MA);
      if (gp >= g0 && gp < g0 + k) h.tmask |= 1u << i;
    }
    h.ntargets = k;
    gs.push_back(h);
    g0 += k;
  }
  return gs;
}

// complex64 cluster-pair groups (lrq_sweep_wdc.cuh): for n - 13 in [16, 20]
// the qubits above group A split into two groups of 8-10 targets whose
// 128 KB tiles (two CTAs) have 128-512 B runs, instead of 64 / 128 B runs in
// 64 KB tiles.  The group with the longer runs takes the top qubits (the
// largest stride).  Opt-in ($LRQ_CLUSTER=1): measured on B200 the longer runs
// do lift the copy ceiling of the tile pattern (5.8 vs 4.6 TB/s), but the
// cluster kernels are issue/latency-bound at 22-24 ms per F sweep against
// 15-16 ms for the single-CTA kernel.
inline bool use_cluster_plan(int n, int pair) {
  const char* v = getenv("LRQ_CLUSTER");
  if (!(v && *v == '1')) return false;
  const int rest = n - (kUnitBits + pair);
  return pair == 1 && rest >= 16 && rest <= 20;
}
inline std::vector<PlanGroup> plan_groups_cluster(int n, int pair) {
  const int KA = kUnitBits + pair;
  std::vector<PlanGroup> gs;
  PlanGroup a;
  a.kind = GK_A;
  a.m = KA;
  a.q0 = KA;
  a.tmask = (1u << KA) - 1u;
  a.ntargets = KA;
  gs.push_back(a);
  const int rest = n - KA;
  const int k_lo = rest / 2, k_hi = rest - k_lo;  // k_hi >= k_lo: more targets low, longer runs on top
  const int ks[2] = {k_hi, k_lo};
  int q = KA;
  for (int k : ks) {
    PlanGroup h;
    h.kind = k == 10 ? GK_C10 : (k == 9 ? GK_C9 : GK_C8);
    h.m = group_ma(h.kind, pair);  // = 14 - k
    h.q0 = q;
    h.tmask = ((1u << KA) - 1u) & ~((1u << h.m) - 1u);  // the k - 1 local targets
    h.ntargets = k;
    h.cross = q + k - 1;
    gs.push_back(h);
    q += k;
  }
  return gs;
}

// Butterfly masks come from the compile-time programs (prog_mask); a masked
// register bit that is not one of the group's targets gets tangent 0.
// mask*[r] = register amp bits that take a real butterfly in round r,
// tmask*[r] = the same bits as tile amp bits.
// warp-decoupled program (high groups; P, M, F sweeps): layout L1 holds tile
// unit bits 7..11 in registers, L2 unit bits 2..6; rounds M: L1, L2;
// F: L1 (mix1), L2 (mix1, phase, mix2), L1 (mix2).  Register unit bit k
// (tile amp bit (L1 ? 7 : 2) + k + pair) takes tangent SweepParams::tf[w][r][k].
// P (no load): L2 (phase, mix2), L1 (mix2).
inline int wd_layout(int kind, int r) {
  if (kind == SK_P) return r == 0 ? 2 : 1;
  return (kind == SK_F && r == 1) || (kind == SK_M && r == 1) ? 2 : 1;
}
inline void plan_rounds_wd(const PlanGroup& g, int pair, PlanSweep& sw) {
  sw.nrounds = sw.kind == SK_F ? 3 : 2;  // M, P: 2
  const unsigned targets[2] = {sw.target1 ? sw.target1 : g.tmask, g.tmask};
  if (!sw.ntarget1) sw.ntarget1 = sw.target1 ? __builtin_popcount(sw.target1) : g.ntargets;
  if (!sw.ntarget2) sw.ntarget2 = g.ntargets;
  for (int r = 0; r < sw.nrounds; ++r) {
    const int L = wd_layout(sw.kind, r);
    const bool mixes[2] = {sw.kind == SK_M || (sw.kind == SK_F && r < 2), (sw.kind == SK_F && r >= 1) || sw.kind == SK_P};
    unsigned m[2] = {0, 0}, tm[2] = {0, 0};
    for (int w = 0; w < 2; ++w)
      for (int k = 0; k < 5; ++k) {  // register unit bit k = unit bit (L1 ? 7 : 2) + k
        const unsigned tb = 1u << ((L == 1 ? 7 : 2) + k + pair);
        if (mixes[w] && (targets[w] & tb)) {
          m[w] |= 1u << k;  // tangent slot k (the complex64 pair bit never mixes)
          tm[w] |= tb;
        }
      }
    sw.mask1[r] = sw.beta1 >= 0 ? m[0] : 0;
    sw.mask2[r] = sw.beta2 >= 0 ? m[1] : 0;
    sw.tmask1[r] = sw.beta1 >= 0 ? tm[0] : 0;
    sw.tmask2[r] = sw.beta2 >= 0 ? tm[1] : 0;
  }
}

inline void plan_rounds(const PlanGroup& g, int pair, PlanSweep& sw) {
  if (sw.prog == 1 || sw.prog == 2) {
    plan_rounds_wd(g, pair, sw);
    return;
  }
  const int RA = 4 + pair;
  sw.nrounds = prog_rounds(g.kind, pair, sw.kind);
  const unsigned targets[2] = {sw.target1 ? sw.target1 : g.tmask, g.tmask};
  if (!sw.ntarget1) sw.ntarget1 = sw.target1 ? __builtin_popcount(sw.target1) : g.ntargets;
  if (!sw.ntarget2) sw.ntarget2 = g.ntargets;
  for (int r = 0; r < sw.nrounds; ++r) {
    const int lo = prog_lo(g.kind, pair, sw.kind, r);
    const unsigned pm[2] = {prog_mask(g.kind, pair, sw.kind, r, 0), prog_mask(g.kind, pair, sw.kind, r, 1)};
    unsigned m[2] = {0, 0}, tm[2] = {0, 0};
    for (int w = 0; w < 2; ++w)
      for (int a = 0; a < RA; ++a) {
        const unsigned tb = 1u << reg_tile_bit(pair, lo, a);
        if (((pm[w] >> a) & 1u) && (targets[w] & tb)) {
          m[w] |= 1u << a;
          tm[w] |= tb;
        }
      }
    sw.mask1[r] = sw.beta1 >= 0 ? m[0] : 0;
    sw.mask2[r] = sw.beta2 >= 0 ? m[1] : 0;
    sw.tmask1[r] = sw.beta1 >= 0 ? tm[0] : 0;
    sw.tmask2[r] = sw.beta2 >= 0 ? tm[1] : 0;
  }
}

// global qubit behind tangent slot a of round r (the bit a of mask1/mask2)
inline int sweep_qubit(const PlanGroup& g, const PlanSweep& w, int pair, int r, int a) {
  const int tb = w.prog >= 1 ? (wd_layout(w.kind, r) == 1 ? 7 : 2) + a + pair
                             : reg_tile_bit(pair, prog_lo(g.kind, pair, w.kind, r), a);
  return tb < g.m ? tb : g.q0 + (tb - g.m);
}

inline PlanSweep make_sweep(int group, int kind, int b1, int ph, int b2, bool red) {
  PlanSweep s;
  s.group = group;
  s.kind = kind;
  s.beta1 = b1;
  s.phase = ph;
  s.beta2 = b2;
  s.reduce = red;
  s.nrounds = 0;
  s.target1 = 0;
  s.ntarget1 = s.ntarget2 = 0;
  s.remap_after = false;
  s.perm = 0;
  s.prog = 0;
  for (int r = 0; r < kMaxRounds; ++r) s.mask1[r] = s.mask2[r] = s.tmask1[r] = s.tmask2[r] = 0;
  return s;
}

inline Plan make_plan(int n, int pair, int p) {
  Plan P;
  P.n = n;
  P.pair = pair;
  P.KA = kUnitBits + pair;
  P.small = n < P.KA;
  if (P.small || p < 1) return P;
  const bool cluster = use_cluster_plan(n, pair);
  P.groups = cluster ? plan_groups_cluster(n, pair) : plan_groups(n, pair);
  const int S = (int)P.groups.size();
  if (S >= 3) {
    // >= 2 high groups: the fused F sweeps go to the two end HIGH groups
    // (warp-decoupled kernel, two transposes), group A sits in
    // the middle (M sweeps) and takes the final reduction: the last layer
    // visits its remaining groups with A last.
    //   order  E1=G_1, mids = A, G_2..G_{S-2}, E2 = G_{S-1}
    std::vector<int> seq;
    seq.push_back(1);
    seq.push_back(0);
    for (int i = 2; i < S - 1; ++i) seq.push_back(i);
    seq.push_back(S - 1);
    // the last layer enters one end group through an F and mixes the other
    // end with a plain M: let that M fall on the cheaper (H4: 128 B runs) end
    {
      const int first_last = (p == 1 || (p - 2) % 2 == 1) ? seq.front() : seq.back();
      const int other = first_last == seq.front() ? seq.back() : seq.front();
      // (longer runs stream faster: H4 over H, C9 over C10)
      if (P.groups[other].m < P.groups[first_last].m) std::reverse(seq.begin(), seq.end());
    }
    const char* nowd = getenv("LRQ_NO_WD");  // debugging: classic kernels, same order
    auto wd = [&](int gi, int kind) {
      // cluster groups: every sweep on the cluster-pair kernel (prog 2)
      if (is_cluster_group(P.groups[gi].kind)) return 2;
      // F only: a lone high-group M (last layer) streams faster on the classic TMA kernel
      return !(nowd && *nowd == '1') && P.groups[gi].kind != GK_A && (kind == SK_F || kind == SK_P) ? 1 : 0;
    };
    auto push = [&](int gi, int kind, int b1, int ph, int b2, bool red) {
      PlanSweep w = make_sweep(gi, kind, b1, ph, b2, red);
      w.prog = wd(gi, kind);
      P.sweeps.push_back(w);
    };
    // layer k (< p-1) visits seq forward for even k, backward for odd k; its
    // last group is layer k+1's first (one F sweep); layer p-1 visits the
    // groups it has left with A last (R)
    auto layer_order = [&](int k) {
      std::vector<int> o(seq);
      if (k % 2) std::reverse(o.begin(), o.end());
      return o;
    };
    for (int k = 0; k < p; ++k) {
      std::vector<int> o = layer_order(k);
      if (k == p - 1) {
        // keep o[0] first (entered by the previous F, or P), put A last
        std::vector<int> rest;
        for (size_t i = 1; i < o.size(); ++i)
          if (o[i] != 0) rest.push_back(o[i]);
        rest.push_back(0);
        o.resize(1);
        o.insert(o.end(), rest.begin(), rest.end());
      }
      if (k == 0) push(o[0], SK_P, -1, 0, 0, false);
      for (size_t i = 1; i + 1 < o.size(); ++i) push(o[i], SK_M, k, -1, -1, false);
      if (k + 1 < p) push(o.back(), SK_F, k, k + 1, k + 1, false);
      else push(o.back(), SK_R, k, -1, -1, true);
    }
    for (PlanSweep& w : P.sweeps) plan_rounds(P.groups[w.group], pair, w);
    return P;
  }
  if (S == 1) {
    P.sweeps.push_back(make_sweep(0, SK_P, -1, 0, 0, false));
    for (int k = 1; k < p; ++k) P.sweeps.push_back(make_sweep(0, SK_L, -1, k, k, k == p - 1));
    if (p == 1) P.sweeps.push_back(make_sweep(0, SK_Q, -1, -1, -1, true));
  } else {
    // layer k visits groups backward when (p-1-k) is even, so layer p-1 ends on G_1
    auto order = [&](int k, int i) { return ((p - 1 - k) % 2 == 0) ? S - 1 - i : i; };
    P.sweeps.push_back(make_sweep(order(0, 0), SK_P, -1, 0, 0, false));
    for (int k = 0; k < p; ++k) {
      for (int i = 1; i < S - 1; ++i) P.sweeps.push_back(make_sweep(order(k, i), SK_M, k, -1, -1, false));
      const int last = order(k, S - 1);
      if (k + 1 < p) P.sweeps.push_back(make_sweep(last, SK_F, k, k + 1, k + 1, false));
      else P.sweeps.push_back(make_sweep(last, SK_R, k, -1, -1, true));
    }
  }
  for (PlanSweep& s : P.sweeps) plan_rounds(P.groups[s.group], pair, s);
  return P;
}

// ---------------------------------------------------------------------------
// Distributed plan (one process per GPU, G = 2^g ranks, n_loc = n - g local
// qubits).  Physical bits [0, n_loc) are local, [n_loc, n) are
// the rank.  The cost phase is fully local (the rank's qubits enter as a field
// and a constant), the mixer needs every qubit local once per layer: after a
// layer's local sweeps one remap (all-to-all block transpose) swaps the g
// global qubits with the top g local bits L' (inside the last group Z), and
// the next sweep on Z starts with the mixer of the just-arrived qubits:
//   layer 0:  P(Z) [init, phase_0, mix_0(Z)], M(others) mix_0, REMAP
//   layer k:  F(Z) [mix_{k-1}(L'), phase_k, mix_k(Z)], M(others) mix_k, REMAP
//   end:      M(Z) [mix_{p-1}(L')], Q(A) in the permutation the layers left
// Each sweep records the permutation state it runs in (the phase terms
// depend on it); two remaps restore the identity.
inline Plan make_dist_plan(int n_loc, int g, int pair, int p) {
  Plan P;
  P.n = n_loc;
  P.pair = pair;
  P.KA = kUnitBits + pair;
  P.small = false;
  P.groups = plan_groups(n_loc, pair);
  const int S = (int)P.groups.size();
  const int Z = S - 1;
  // the remap swaps the top g local qubits L' into the rank bits, so all of
  // L' must be targets of Z.  A short last group (fewer than g targets) takes
  // the missing ones from the top of the group below: its tile slid down to
  // the top of the range and already holds them as non-target bits.
  if (S >= 2 && P.groups[Z].ntargets < g) {
    PlanGroup& z = P.groups[Z];
    PlanGroup& y = P.groups[Z - 1];
    const int lo = n_loc - g, hi = n_loc - z.ntargets;  // qubits [lo, hi) move from y to z
    for (int i = 0; i < P.KA; ++i) {
      const int gy = i < y.m ? i : y.q0 + (i - y.m);
      if (gy >= lo && gy < hi && ((y.tmask >> i) & 1u)) y.tmask &= ~(1u << i);
      const int gz = i < z.m ? i : z.q0 + (i - z.m);
      if (i >= z.m && gz >= lo && gz < hi) z.tmask |= 1u << i;
    }
    y.ntargets -= hi - lo;
    z.ntargets += hi - lo;
  }
  const PlanGroup& gz = P.groups[Z];
  // tile bits of group Z holding the top g local qubits L'
  unsigned lmask = 0;
  for (int i = gz.m; i < P.KA; ++i) {
    const int gp = gz.q0 + (i - gz.m);
    if (gp >= n_loc - g && gp < n_loc) lmask |= 1u << i;
  }
  int perm = 0;
  for (int k = 0; k < p; ++k) {
    PlanSweep z = k == 0 ? make_sweep(Z, SK_P, -1, 0, 0, false) : make_sweep(Z, SK_F, k - 1, k, k, false);
    if (k > 0) z.target1 = lmask;
    z.perm = perm;
    P.sweeps.push_back(z);
    for (int o = Z - 1; o >= 0; --o) {  // group A last: its contiguous tiles can carry the remap
      PlanSweep m = make_sweep(o, SK_M, k, -1, -1, false);
      m.perm = perm;
      P.sweeps.push_back(m);
    }
    P.sweeps.back().remap_after = true;
    perm ^= 1;
  }
  PlanSweep last = make_sweep(Z, SK_M, p - 1, -1, -1, false);
  last.target1 = lmask;
  last.perm = perm;
  P.sweeps.push_back(last);
  // the final pass runs in whichever permutation the layers left (an odd p
  // leaves the global and top local qubits swapped): no restoring remap.
  // Reductions, max-cut argmin and the sampler map indices through the
  // permutation; amplitude reads restore the identity layout on demand
  // (lrq_restore_layout).
  PlanSweep q = make_sweep(0, SK_Q, -1, -1, -1, true);
  q.perm = perm;
  P.sweeps.push_back(q);
  // P and F sweeps of the (high) group Z run the warp-decoupled kernel
  const char* nowd = getenv("LRQ_NO_WD");
  for (PlanSweep& s : P.sweeps)
    if (!(nowd && *nowd == '1') && P.groups[s.group].kind != GK_A && (s.kind == SK_P || s.kind == SK_F)) s.prog = 1;
  for (PlanSweep& s : P.sweeps) plan_rounds(P.groups[s.group], pair, s);
  return P;
}

inline std::string plan_json(const Plan& P) {
  static const char* kinds = "PMFRLQN";
  std::string s = "{\"n\":" + std::to_string(P.n) + ",\"K\":" + std::to_string(P.KA) + ",\"pair\":" +
                  std::to_string(P.pair) + ",\"small\":" + (P.small ? "true" : "false") + ",\"groups\":[";
  for (size_t i = 0; i < P.groups.size(); ++i) {
    const PlanGroup& g = P.groups[i];
    s += (i ? "," : "");
    const char* kn = g.kind == GK_A ? "A" : g.kind == GK_H4 ? "H4" : g.kind == GK_C10 ? "C10" : g.kind == GK_C9 ? "C9"
                     : g.kind == GK_C8 ? "C8" : "H";
    s += "{\"kind\":\"" + std::string(kn) + "\",\"m\":" + std::to_string(g.m) + ",\"q0\":" + std::to_string(g.q0) +
         ",\"tmask\":" + std::to_string(g.tmask) + ",\"cross\":" + std::to_string(g.cross) + "}";
  }
  s += "],\"sweeps\":[";
  for (size_t i = 0; i < P.sweeps.size(); ++i) {
    const PlanSweep& w = P.sweeps[i];
    const PlanGroup& g = P.groups[w.group];
    s += (i ? "," : "");
    s += "{\"group\":" + std::to_string(w.group) + ",\"kind\":\"" + kinds[w.kind] + "\",\"init\":" +
         (w.kind == SK_P ? "true" : "false") + ",\"beta1\":" + std::to_string(w.beta1) +
         ",\"phase\":" + std::to_string(w.phase) + ",\"beta2\":" + std::to_string(w.beta2) +
         ",\"reduce\":" + (w.reduce ? "true" : "false") + ",\"rounds\":[";
    for (int r = 0; r < w.nrounds; ++r) {
      s += (r ? "," : "");
      if (w.prog >= 1) {  // lo: the lowest register unit bit of the layout
        const bool ph = (w.kind == SK_F && r == 1) || (w.kind == SK_P && r == 0);
        s += "[" + std::to_string(wd_layout(w.kind, r) == 1 ? 7 : 2) + "," + std::to_string(w.tmask1[r]) + "," +
             std::to_string(w.tmask2[r]) + "," + (ph ? "1" : "0") + ",0]";
        continue;
      }
      s += "[" + std::to_string(prog_lo(g.kind, P.pair, w.kind, r)) + "," + std::to_string(w.tmask1[r]) + "," +
           std::to_string(w.tmask2[r]) + "," + (prog_phase(w.kind, g.kind, P.pair, r) ? "1" : "0") + "," +
           (prog_reduce(w.kind, g.kind, P.pair, r) ? "1" : "0") + "]";
    }
    s += "],\"prog\":" + std::to_string(w.prog) + "}";
  }
  s += "]}";
  return s;
}

}  // namespace lrq
