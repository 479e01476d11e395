// The tiled sweep kernel (v2): one HBM round trip of the state applies, to
// every tile of 4096 16-byte units (2^13 complex64 / 2^12 complex128
// amplitudes), a compile-time program of
//     [init | load] [mixer 1] [cost phase] [mixer 2] [reductions] [store]
// (DESIGN.md §3.2).  Each of the 256 threads keeps 16 units in registers; the
// butterflies of the qubits held in registers run there, and shared memory
// (padded: unit c lives at c + c/16, conflict-free for every layout) only
// transposes the tile between register layouts ("rounds").
//
// Reference operations fused here (lrqbench):
//   RZZ per edge  engine.py:147-155  -> exp(-i E_J(z)), E_J assembled per tile
//   RX per qubit  engine.py:137-144  -> scaled butterfly x + i t y (FFMA2 on c64)
//   H layer       engine.py:128-134  -> init value v_n (no load at all)
//   probabilities / expected_r / cut_values_range  engine.py:94-96,214-226,
//                 problem.py:158-171 -> per-tile sum p, sum p*E_w, min E_w
//
// Index spaces.  Amplitude z has qubit k at bit k.  A complex64 unit holds
// the amplitude pair (z, z^1) ("pair bit" = amp bit 0, always in registers);
// a complex128 unit holds one amplitude.  Tile amp bit i maps to global amp
// bit g(i) = i < MA ? i : q0 + (i - MA): group A (MA = KA) is one contiguous
// run; a high group H is 2^(KA-MA) runs of 2^MA amplitudes (64 B / 256 B).
// A layout "lo" puts tile unit bits [lo, lo+4) in registers; the thread index
// fills the remaining 8 unit bits in ascending order.
#pragma once
#include <cuda.h>

#include "lrq_device.cuh"

namespace lrq {

constexpr int kMaxRounds = 8;
constexpr int kUnitBits = 12;  // units per tile = 4096
constexpr int kThreads = 256;  // 8 thread bits + 4 register unit bits

// A: tile = one contiguous run.  H: runs of 2^MA amplitudes, MA = 3 (c64,
// 64 B) or 4 (c128, 256 B).  H4: complex64 runs of 16 amplitudes (128 B) for
// the middle groups, which take a mixer-only sweep every layer: whole 128 B
// lines keep twice the bytes in flight per outstanding L2 request.
enum GroupKind {
  GK_A = 0,
  GK_H = 1,
  GK_H4 = 2,
  // complex64 cluster-pair groups (lrq_sweep_wdc.cuh): a 128 KB tile over two
  // CTAs, k targets with runs of 2^(14-k) amplitudes (C10: 128 B, C9: 256 B,
  // C8: 512 B); the top target is the cross qubit between the two CTAs
  GK_C10 = 3,
  GK_C9 = 4,
  GK_C8 = 5
};
__host__ __device__ constexpr bool is_cluster_group(int gk) { return gk >= GK_C10; }
enum SweepKind {
  SK_P = 0,  // init, phase, mixer 2                         (first sweep)
  SK_M = 1,  // load, mixer 1, store                         (middle sweeps)
  SK_F = 2,  // load, mixer 1, phase, mixer 2, store         (layer boundary)
  SK_R = 3,  // load, mixer 1, reductions, store             (last sweep, group A)
  SK_L = 4,  // load, phase, mixer 2 [, reductions], store   (single-group plans)
  SK_Q = 5,  // load, reductions                             (recompute, group A)
  SK_N = 6   // reductions over E only, no state             (max-cut search)
};

// ---------------------------------------------------------------------------
// compile-time round programs (shared with the host planner)

__host__ __device__ constexpr int num_layouts(int gk, int pair) { return gk == GK_A ? 3 : (pair ? 3 : 2); }
__host__ __device__ constexpr int layout_lo(int gk, int pair, int i) {
  // A: {8, 0, 4}; H: {8, 4, 2} (c64, runs of 8 amps) / {8, 4} (c128, runs of 16 amps);
  // H4 (c64, runs of 16 amps): {8, 4, 3}
  return gk == GK_A ? (i == 0 ? 8 : (i == 1 ? 0 : 4)) : (i == 0 ? 8 : (i == 1 ? 4 : (gk == GK_H4 ? 3 : 2)));
}
__host__ __device__ constexpr int group_ma(int gk, int pair) {
  return gk == GK_A ? 12 + pair
         : gk == GK_C10 ? 4
         : gk == GK_C9  ? 5
         : gk == GK_C8  ? 6
                        : (gk == GK_H4 ? 4 : (pair ? 3 : 4));
}

__host__ __device__ constexpr int prog_rounds(int gk, int pair, int sk) {
  return sk == SK_F ? 2 * num_layouts(gk, pair) - 1 : ((sk == SK_Q || sk == SK_N) ? 1 : num_layouts(gk, pair));
}
// layout index of round r
__host__ __device__ constexpr int prog_layout(int gk, int pair, int sk, int r) {
  return (sk == SK_P || sk == SK_L) ? num_layouts(gk, pair) - 1 - r
         : sk == SK_F               ? (r < num_layouts(gk, pair) ? r : 2 * num_layouts(gk, pair) - 2 - r)
         : (sk == SK_Q || sk == SK_N) ? 0
                                      : r;
}
__host__ __device__ constexpr int prog_lo(int gk, int pair, int sk, int r) {
  return layout_lo(gk, pair, prog_layout(gk, pair, sk, r));
}
__host__ __device__ constexpr bool prog_m1(int sk, int gk, int pair, int r) {
  return (sk == SK_M || sk == SK_R) || (sk == SK_F && r < num_layouts(gk, pair));
}
__host__ __device__ constexpr bool prog_m2(int sk, int gk, int pair, int r) {
  return (sk == SK_P || sk == SK_L) || (sk == SK_F && r >= num_layouts(gk, pair) - 1);
}
__host__ __device__ constexpr bool prog_phase(int sk, int gk, int pair, int r) {
  return ((sk == SK_P || sk == SK_L) && r == 0) || (sk == SK_F && r == num_layouts(gk, pair) - 1);
}
__host__ __device__ constexpr bool prog_reduce(int sk, int gk, int pair, int r) {
  return ((sk == SK_R || sk == SK_L) && r == prog_rounds(gk, pair, sk) - 1) || sk == SK_Q || sk == SK_N;
}
__host__ __device__ constexpr int prog_store_lo(int gk, int pair, int sk) {
  return prog_lo(gk, pair, sk, prog_rounds(gk, pair, sk) - 1);
}
// register amp bit a of layout lo -> tile amp bit
__host__ __device__ constexpr int reg_tile_bit(int pair, int lo, int a) { return pair ? (a == 0 ? 0 : lo + a) : lo + a; }
// thread index bit j of layout lo -> tile amp bit
__host__ __device__ constexpr int thr_tile_bit(int pair, int lo, int j) { return (j < lo ? j : j + 4) + pair; }
// tile amp bits that can be mixer targets: all of group A, the run-index bits of H
__host__ __device__ constexpr int first_target(int gk, int pair) { return gk == GK_A ? 0 : group_ma(gk, pair); }
__host__ __device__ constexpr bool prog_mixes(int sk, int gk, int pair, int r, int w) {
  return w == 0 ? prog_m1(sk, gk, pair, r) : prog_m2(sk, gk, pair, r);
}
// compile-time butterfly mask (over register amp bits a < 4+pair) of round r
// for mixer w: the potential targets not already visited by that mixer in an
// earlier round.  Non-target bits of a short H group get a zero angle at run
// time instead (x + i*0*y = x), so every mask is static.
__host__ __device__ constexpr unsigned prog_mask(int gk, int pair, int sk, int r, int w) {
  unsigned done = 0;
  for (int q = 0; q < r; ++q)
    if (prog_mixes(sk, gk, pair, q, w))
      for (int a = 0; a < 4 + pair; ++a) done |= 1u << reg_tile_bit(pair, prog_lo(gk, pair, sk, q), a);
  if (!prog_mixes(sk, gk, pair, r, w)) return 0u;
  unsigned m = 0;
  for (int a = 0; a < 4 + pair; ++a) {
    const int tb = reg_tile_bit(pair, prog_lo(gk, pair, sk, r), a);
    if (tb >= first_target(gk, pair) && !((done >> tb) & 1u)) m |= 1u << a;
  }
  return m;
}

struct MatArg {
  const double* M;    // n*n symmetric, zero diagonal, physical bit order
  const double* ext;  // n: field from bits outside this shard (global qubits)
  double cst;         // constant from bits outside this shard
};

struct SweepParams {
  // H groups: 5-D tensor map over the tile's 2^(KA-MA) runs, used to prefetch
  // a CTA's next tile into L2 with one TMA instruction (has_tmap = 0: none)
  CUtensorMap tmap;
  int has_tmap;
  int nstages;  // TMA path: shared-memory stages in the load ring (2 or 3)
  void* amps;
  int n;   // local amp bits
  int q0;  // global amp bit of tile amp bit MA (group A: KA)
  long long num_tiles;
  int reduce;  // SK_L: reduce in the last round
  // butterfly tangent per [mixer][round][register amp bit] (0 for non-targets)
  float tf[2][kMaxRounds][5];
  double td[2][kMaxRounds][5];
  double scale_re, scale_im;  // product of the per-qubit mixer factors
  double init_re, init_im;
  MatArg J, W;
  int min_bit;  // local amp bit that must be 0 in the min-E search (-1 none, -2 skip all)
  double* red_p;
  double* red_pE;
  double* red_minE;
  unsigned long long* red_arg;
  double* red_maxE;  // per-tile max E (may be null)
  int search;        // reductions: 1 = also min E with argmin (max-cut search) and max E
  double tc[2];      // cluster groups: mixer tangents of the cross qubit (mixer 1, mixer 2; 0 = none)
  // p-weighted energy histogram (may be null): bin b = floor((E - hist_lo) *
  // hist_scale) clamped to [0, hist_bins); each amplitude adds round(p 2^60)
  // to its bin as a 64-bit integer, so the totals do not depend on the order
  // (deterministic) and sum to 2^60 sum p
  unsigned long long* hist;
  int hist_bins;
  double hist_lo, hist_scale;
  // fused remap (distributed plans, group-A M sweep before a remap): the tiles
  // of block b (top g local bits; 2^rbits tiles each) are stored straight
  // into rdst[b], rank b's next state buffer at this rank's block (peer
  // memory over NVLink) instead of in place
  int remap;
  int rbits;
  void* rdst[8];
  int wd_prefetch;  // warp-decoupled sweeps: L2 prefetch of the tile this many ahead at each refill (0: off)
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }
constexpr int kTileUnitsPadded = (1 << kUnitBits) + (1 << (kUnitBits - 4));

// dynamic shared memory of sweep_kernel
__host__ __device__ inline size_t sweep_smem_bytes(int n, bool amps, bool usesJ, bool usesW, int hist_bins = 0) {
  size_t b = amps ? 16 * (size_t)kTileUnitsPadded : 0;
  if (usesJ) b = align16(b + 8 * (size_t)(n * n + n));
  if (usesW) b = align16(b + 8 * (size_t)(n * n + n));
  b += 8 * (size_t)(2 * 2 * 16 + 4);    // hB[parity][mat][16], EBB[parity][mat]
  b += 8 * (size_t)(2 * 6 * kThreads);  // per-thread constants [mat][RA+1][thread]
  b = align16(b);
  b += 16 * 32 + 8 * 32 + 8 * 32;  // PRR[32] (c128), PRR32[32] (c64), ERR[32]
  b += 8 * 5 * (kThreads / 32);  // reduction scratch
  b += 8 * (size_t)hist_bins;     // shared energy histogram
  return align16(b);
}


template <typename T>
struct UnitT;
template <>
struct UnitT<float> {
  typedef float4 U;
  typedef float2 A;
  static constexpr int PAIR = 1;
};
template <>
struct UnitT<double> {
  typedef double2 U;
  typedef double2 A;
  static constexpr int PAIR = 0;
};

// amplitude v of the register file (compile-time v -> register moves)
__device__ __forceinline__ float2 amp_get(const float4 (&r)[16], int v) {
  const float4& q = r[v >> 1];
  return (v & 1) ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
}
__device__ __forceinline__ void amp_set(float4 (&r)[16], int v, float2 a) {
  float4& q = r[v >> 1];
  if (v & 1) {
    q.z = a.x;
    q.w = a.y;
  } else {
    q.x = a.x;
    q.y = a.y;
  }
}
__device__ __forceinline__ double2 amp_get(const double2 (&r)[16], int v) { return r[v]; }
__device__ __forceinline__ void amp_set(double2 (&r)[16], int v, double2 a) { r[v] = a; }

__host__ __device__ constexpr int phys(int c) { return c + (c >> 4); }

template <typename T, int GK, int SK>
struct SweepCtx {
  typedef typename UnitT<T>::U U;
  typedef typename UnitT<T>::A A;
  static constexpr int PAIR = UnitT<T>::PAIR;
  static constexpr int RA = 4 + PAIR;  // register amp bits
  static constexpr int NV = 1 << RA;
  static constexpr int KA = kUnitBits + PAIR;
  static constexpr int MA = group_ma(GK, PAIR);
  static constexpr int MU = MA - PAIR;  // coalescing unit bits
  static constexpr int NR = prog_rounds(GK, PAIR, SK);

  __device__ static __forceinline__ int gpos(int i, int q0) { return i < MA ? i : q0 + (i - MA); }
  __device__ static __forceinline__ bool blockbit(int j, int q0) { return j >= MA && !(j >= q0 && j < q0 + KA - MA); }
  __device__ static __forceinline__ int ebase(int t, int lo) { return (t & ((1 << lo) - 1)) | ((t >> lo) << (lo + 4)); }
  // global unit index of tile unit e (relative to the tile base)
  __device__ static __forceinline__ uint64_t gunit(int e, int qU) {
    return (uint64_t)(e & ((1 << MU) - 1)) | ((uint64_t)(e >> MU) << qU);
  }
  __device__ static __forceinline__ int gshift(int lo, int qU) { return lo >= MU ? lo - MU + qU : lo; }

  // per-thread constants of layout lo for matrix M: T_a (a < RA) and E_TT
  __device__ static void thread_consts(const double* M, int n, int q0, int lo, int t, double* dst) {
    for (int a = 0; a < RA; ++a) {
      const int ga = gpos(reg_tile_bit(PAIR, lo, a), q0);
      double acc = 0.0;
      for (int j = 0; j < 8; ++j) {
        const double w = M[ga * n + gpos(thr_tile_bit(PAIR, lo, j), q0)];
        acc += ((t >> j) & 1) ? -w : w;
      }
      dst[a * kThreads + t] = acc;
    }
    double ett = 0.0;
    for (int j = 0; j < 8; ++j) {
      const int gj = gpos(thr_tile_bit(PAIR, lo, j), q0);
      const double sj = ((t >> j) & 1) ? -1.0 : 1.0;
      for (int j2 = j + 1; j2 < 8; ++j2) {
        const double w = M[gj * n + gpos(thr_tile_bit(PAIR, lo, j2), q0)];
        ett += (((t >> j2) & 1) ? -sj : sj) * w;
      }
    }
    dst[RA * kThreads + t] = ett;
  }

  // energy among the register bits for pattern v
  __device__ static double err_entry(const double* M, int n, int q0, int lo, int v) {
    double acc = 0.0;
    for (int a = 0; a < RA; ++a) {
      const int ga = gpos(reg_tile_bit(PAIR, lo, a), q0);
      const double sa = ((v >> a) & 1) ? -1.0 : 1.0;
      for (int b = a + 1; b < RA; ++b) {
        const double w = M[ga * n + gpos(reg_tile_bit(PAIR, lo, b), q0)];
        acc += (((v >> b) & 1) ? -sa : sa) * w;
      }
    }
    return acc;
  }

  // per-tile field on every tile bit from the tile's fixed bits (warp w0) and
  // the fixed bits' own energy (warp w0+1)
  __device__ static void block_consts(const double* M, const double* X, double cst, int n, int q0, uint64_t base,
                                      int w0, double* hb, double* ebb, int tl) {
    const int warp = tl >> 5, lane = tl & 31;  // tl: thread index within the 256-thread team
    // the block bits are [MA, q0) and [q0 + KA - MA, n), visited in ascending
    // order (the same sums as a full j loop that skips the tile bits, without
    // a branch per bit)
    const int lo_end = q0 < n ? q0 : n, hi_beg = q0 + KA - MA > MA ? q0 + KA - MA : MA;
    if (warp == w0) {
      if (lane < KA) {
        const int gi = gpos(lane, q0);
        const double* Mi = M + gi * n;
        double acc = X[gi];
#pragma unroll 4
        for (int j = MA; j < lo_end; ++j) acc += Mi[j] * spin(base, j);
#pragma unroll 4
        for (int j = hi_beg; j < n; ++j) acc += Mi[j] * spin(base, j);
        hb[lane] = acc;
      }
    } else if (warp == w0 + 1) {
      double term = 0.0;
      for (int j = lane; j < n; j += 32) {
        if (!blockbit(j, q0)) continue;
        const double* Mj = M + j * n;
        double f = 0.0;
#pragma unroll 4
        for (int l = MA; l < lo_end; ++l) f += Mj[l] * spin(base, l);
#pragma unroll 4
        for (int l = hi_beg; l < n; ++l) f += Mj[l] * spin(base, l);
        term += spin(base, j) * (X[j] + 0.5 * f);
      }
      for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
      if (lane == 0) *ebb = cst + term;
    }
  }

  // ---- register-file butterflies: amp pairs (v, v | 1<<b) for b in MASK ----
  // (x, y) <- (x + i t y, y + i t x): RX up to the per-qubit scalar folded
  // into SweepParams::scale; t = 0 leaves a non-target bit untouched.
  template <unsigned MASK>
  __device__ static __forceinline__ void mix(U (&r)[16], const float* tf, const double* td) {
#pragma unroll
    for (int b = 0; b < RA; ++b) {
      if (!((MASK >> b) & 1u)) continue;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if ((v >> b) & 1) continue;
        const int w = v | (1 << b);
        const A x = amp_get(r, v), y = amp_get(r, w);
        if constexpr (PAIR) {
          const float2 tv = make_float2(-tf[b], tf[b]);
          amp_set(r, v, bf_half(x, y, tv));
          amp_set(r, w, bf_half(y, x, tv));
        } else {
          amp_set(r, v, bf_half(x, y, td[b]));
          amp_set(r, w, bf_half(y, x, td[b]));
        }
      }
    }
  }

  template <int LO>
  __device__ static __forceinline__ void to_smem(U* tile, const U (&r)[16], int t) {
    U* p = tile + phys(ebase(t, LO));
#pragma unroll
    for (int j = 0; j < 16; ++j) p[phys(j << LO)] = r[j];
  }
  template <int LO>
  __device__ static __forceinline__ void from_smem(const U* tile, U (&r)[16], int t) {
    const U* p = tile + phys(ebase(t, LO));
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = p[phys(j << LO)];
  }
  __device__ static __forceinline__ void to_smem_lo(U* tile, const U (&r)[16], int t, int lo) {
    switch (lo) {
      case 0: to_smem<0>(tile, r, t); break;
      case 2: to_smem<2>(tile, r, t); break;
      case 4: to_smem<4>(tile, r, t); break;
      default: to_smem<8>(tile, r, t); break;
    }
  }
  __device__ static __forceinline__ void from_smem_lo(const U* tile, U (&r)[16], int t, int lo) {
    switch (lo) {
      case 0: from_smem<0>(tile, r, t); break;
      case 2: from_smem<2>(tile, r, t); break;
      case 4: from_smem<4>(tile, r, t); break;
      default: from_smem<8>(tile, r, t); break;
    }
  }
};

}  // namespace lrq
