// Warp-decoupled sweeps of a high qubit group (complex64 H: 64 B runs, H4:
// 128 B runs; complex128 H: 256 B runs) for the first (P), mixer-only (M)
// and fused mix -> phase -> mix (F) sweeps.  DESIGN.md §3.2.
//
// A high-group tile is 2^(KA-MA) runs of 2^MA contiguous amplitudes; the run
// bits are NOT mixer targets in this sweep.  Unit bits 0-1 of the tile (inside
// every run) therefore never need a butterfly, and they pick the warp: each
// of the tile's 4 warps owns the 1024 units with its value of those bits and
// exchanges no data with the other three.  Inside a warp the 10 remaining
// unit bits are split 5 lanes x 5 registers (32 16-byte units per thread: 64
// complex64 or 32 complex128 amplitudes), so two layouts cover every target:
//     L1: lane = unit bits 2..6, registers = unit bits 7..11
//     L2: lane = unit bits 7..11, registers = unit bits 2..6
// M = L1 mix, L2 mix; F = L1 mix1, L2 mix1 + phase + mix2, L1 mix2.  Both
// go L1 -> L2 -> L1 through a padded per-warp transpose region (two
// transposes, __syncwarp only), because L1 is the layout whose reads and
// writes of the TMA tile are bank-conflict free.
//
// Per tile: TMA tensor load into a stage (3-stage ring, one full mbarrier
// per stage and team); L1 read; a 4-warp named barrier hands the stage over
// as four 32 x 33-unit transpose regions; at the end a second 4-warp barrier
// pair brackets the write-back in the TMA layout, one thread issues the TMA
// tensor store, waits for it to have read the stage, and loads the tile nst
// steps ahead into it.  Two tiles are in flight per CTA (8 warps, 2 per SM
// sub-partition, which keeps 255 registers for the 32 units a thread holds);
// the two teams run out of phase.  P starts from the H|0> value in L2 and
// loads nothing.
//
// Bank conflicts: the TMA swizzle puts unit e at e ^ ((e >> 3) & SWM); L1
// accesses of the TMA layout have lanes on unit bits 2..4 -> 8 distinct
// 16-byte bank groups per quarter warp; the transposes use slot().
#pragma once
#include "lrq_sweep_tma.cuh"

namespace lrq {

constexpr int kWdTeamsMax = 3;  // tiles in flight per CTA: 2 (M, F: 255 registers) or 3 (P)
constexpr int kWdWarps = 4;     // warps per tile
constexpr int kWdTT = kWdWarps * 32;  // tile threads
constexpr int kWdRAmax = 6;           // register amp bits: (pair) + 5 unit bits
// a stage holds the 64 KB TMA tile plus 2 KB so that, after the tile is read,
// each warp owns a padded 32 x 33-unit transpose region of it
constexpr int kWdStageBytes = 66 * 1024;
constexpr int kWdRegion = 32 * 33;  // units per warp region

__host__ __device__ inline size_t wd_smem_bytes(int n, int nst, bool usesJ) {
  size_t b = (size_t)nst * kWdStageBytes + 128;  // stages + full barriers
  if (usesJ) b = align16(b + 8 * (size_t)(n * n + n));
  b += 8 * (size_t)((kWdRAmax + 1) * kWdTT);  // per-tile-thread constants
  b += 16 * 64;                               // PRR (float2 x 64 or double2 x 32)
  b += 8 * (size_t)(kWdTeamsMax * 20);  // per team: hb[16] fields + 4 warp partials of the block energy
  b += 4 * 64;                         // block-bit list
  return align16(b) + 1024;
}

template <typename T, int GK, int SK>
struct WdSweep {
  typedef typename UnitT<T>::U U;
  static constexpr int PAIR = UnitT<T>::PAIR;
  static_assert(GK == GK_H || ((GK == GK_H4 || is_cluster_group(GK)) && PAIR), "warp-decoupled sweeps serve high groups");
  static constexpr int KA = kUnitBits + PAIR;
  static constexpr int RA = 5 + PAIR;         // register amp bits
  static constexpr int NV = 1 << RA;          // amplitudes per thread
  static constexpr int MA = group_ma(GK, PAIR);  // run amp bits
  static constexpr int MU = MA - PAIR;           // run unit bits (>= 2)
  static constexpr int SWM = (GK == GK_H && PAIR) ? 3 : 7;
  // L2 register bits k hold unit bits 2 + k; those below MU are run bits,
  // never targets: no butterflies for them (H4 c64: bit 2; H c128: bits 2, 3)
  static constexpr unsigned L2MASK = 31u & ~((1u << (MU > 2 ? MU - 2 : 0)) - 1u);
  static constexpr bool PH = SK == SK_F || SK == SK_P;  // has a cost phase
  static constexpr bool INIT = SK == SK_P;              // no load: H|0> value

  __device__ static __forceinline__ int swz(int e) { return e ^ ((e >> 3) & SWM); }
  // unit (a, b) of warp wq: natural TMA position / transposed slot
  __device__ static __forceinline__ int nat(int wq, int a, int b) { return swz(wq | (a << 2) | (b << 7)); }
  // transposed unit (a, b) in the warp's region: row a, column b, rows padded
  // to 33 units -> bank group (a + b) & 7, conflict-free for a lane-a writer
  // and a lane-b reader, and base + immediate addressing both ways
  __device__ static __forceinline__ int slot(int a, int b) { return a * 33 + b; }
  // tile amp bit of register amp bit r in layout L (1: regs = unit bits
  // 7..11, 2: regs = unit bits 2..6); complex64: r = 0 is the pair bit
  __host__ __device__ static constexpr int reg_bit(int L, int r) {
    return PAIR ? (r == 0 ? 0 : (L == 1 ? 7 : 2) + r) : (L == 1 ? 7 : 2) + r;
  }
  // tile amp bit of tile-thread bit j (warp bits = unit bits 0-1, then the 5
  // lane bits)
  __host__ __device__ static constexpr int thr_bit(int L, int j) {
    return PAIR + (j < 2 ? j : (L == 1 ? 2 : 7) + (j - 2));
  }

  __device__ static __forceinline__ int gpos(int i, int q0) { return i < MA ? i : q0 + (i - MA); }

  // butterflies on register unit bits of MASK: (x, y) <- (x + i t y, y + i t x)
  template <unsigned MASK>
  __device__ static __forceinline__ void mix(float4 (&r)[32], const float* tf, const double*) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (!((MASK >> k) & 1u)) continue;
      const float t = tf[k];  // register unit bit k (plan_rounds_wd)
      const float2 tv = make_float2(-t, t);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if ((j >> k) & 1) continue;
        const int w = j | (1 << k);
        const float4 x = r[j], y = r[w];
        const float2 x0 = bf_half(make_float2(x.x, x.y), make_float2(y.x, y.y), tv);
        const float2 x1 = bf_half(make_float2(x.z, x.w), make_float2(y.z, y.w), tv);
        const float2 y0 = bf_half(make_float2(y.x, y.y), make_float2(x.x, x.y), tv);
        const float2 y1 = bf_half(make_float2(y.z, y.w), make_float2(x.z, x.w), tv);
        r[j] = make_float4(x0.x, x0.y, x1.x, x1.y);
        r[w] = make_float4(y0.x, y0.y, y1.x, y1.y);
      }
    }
  }
  template <unsigned MASK>
  __device__ static __forceinline__ void mix(double2 (&r)[32], const float*, const double* td) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (!((MASK >> k) & 1u)) continue;
      const double t = td[k];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if ((j >> k) & 1) continue;
        const int w = j | (1 << k);
        const double2 x = r[j], y = r[w];
        r[j] = bf_half(x, y, t);
        r[w] = bf_half(y, x, t);
      }
    }
  }
  // per-amplitude access of the register file (v: register amp index)
  __device__ static __forceinline__ float2 get(const float4 (&r)[32], int v) {
    return (v & 1) ? make_float2(r[v >> 1].z, r[v >> 1].w) : make_float2(r[v >> 1].x, r[v >> 1].y);
  }
  __device__ static __forceinline__ void set(float4 (&r)[32], int v, float2 a) {
    if (v & 1) {
      r[v >> 1].z = a.x;
      r[v >> 1].w = a.y;
    } else {
      r[v >> 1].x = a.x;
      r[v >> 1].y = a.y;
    }
  }
  __device__ static __forceinline__ double2 get(const double2 (&r)[32], int v) { return r[v]; }
  __device__ static __forceinline__ void set(double2 (&r)[32], int v, double2 a) { r[v] = a; }
  __device__ static __forceinline__ void scale_all(float4 (&r)[32], double2 sc) {
#pragma unroll
    for (int v = 0; v < 64; ++v) set(r, v, cmul_amp(get(r, v), sc));
  }
  __device__ static __forceinline__ void scale_all(double2 (&r)[32], double2 sc) {
#pragma unroll
    for (int v = 0; v < 32; ++v) r[v] = cmul(r[v], sc);
  }

  // cost phase in L2: amplitude v *= sc * exp(-i (C + sum_a s_a F_a + E_RR(v)))
  // (INIT: amplitude v = that phasor); product form as in SweepTile::phase
  __device__ static __forceinline__ void phase(float4 (&r)[32], double C, const double* F, double2 sc,
                                               const void* prr) {
    const float2* PRR32 = reinterpret_cast<const float2*>(prr);
    float2 u[6];
#pragma unroll
    for (int a = 0; a < 6; ++a) u[a] = phasor32(F[a]);
    const float2 eC = cmul32(make_float2((float)sc.x, (float)sc.y), phasor32(C));
    const float2 p01 = cmul32(u[0], u[1]), q01 = cmul32_conj(u[1], u[0]);
    float2 Alo[4];
    Alo[0] = cmul32(eC, p01);
    Alo[1] = cmul32(eC, q01);
    Alo[2] = cmul32_conj(eC, q01);
    Alo[3] = cmul32_conj(eC, p01);
    const float2 p23 = cmul32(u[2], u[3]), q23 = cmul32_conj(u[3], u[2]);
    const float2 Y[4] = {p23, q23, conj32(q23), conj32(p23)};
    const float2 p45 = cmul32(u[4], u[5]), q45 = cmul32_conj(u[5], u[4]);
    const float2 Z[4] = {p45, q45, conj32(q45), conj32(p45)};
#pragma unroll
    for (int h = 0; h < 16; ++h) {
      const float2 Bh = cmul32(Y[h & 3], Z[h >> 2]);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int v = h * 4 + l;
        const float2 ph = cmul32(cmul32(Alo[l], Bh), PRR32[v]);
        set(r, v, INIT ? ph : cmul32(get(r, v), ph));
      }
    }
  }
  __device__ static __forceinline__ void phase(double2 (&r)[32], double C, const double* F, double2 sc,
                                               const void* prr) {
    const double2* PRR = reinterpret_cast<const double2*>(prr);
    const double2 eC = cmul(sc, expmi(C));
    const double2 u0 = expmi(F[0]), u1 = expmi(F[1]), u2 = expmi(F[2]), u3 = expmi(F[3]), u4 = expmi(F[4]);
    const double2 p01 = cmul(u0, u1), q01 = cmul_conj(u1, u0);
    double2 Alo[4];
    Alo[0] = cmul(eC, p01);
    Alo[1] = cmul(eC, q01);
    Alo[2] = cmul_conj(eC, q01);
    Alo[3] = cmul_conj(eC, p01);
    const double2 p23 = cmul(u2, u3), q23 = cmul_conj(u3, u2);
    const double2 Y[4] = {p23, q23, make_double2(q23.x, -q23.y), make_double2(p23.x, -p23.y)};
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const double2 Bh = (h & 4) ? cmul_conj(Y[h & 3], u4) : cmul(Y[h & 3], u4);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int v = h * 4 + l;
        const double2 ph = cmul(cmul(Alo[l], Bh), PRR[v]);
        r[v] = INIT ? ph : cmul(r[v], ph);
      }
    }
  }
};

template <typename T, int GK, int SK, int TEAMS>
__global__ void __launch_bounds__(TEAMS * kWdWarps * 32, 1) sweep_wd_kernel(const __grid_constant__ SweepParams P) {
  typedef WdSweep<T, GK, SK> W;
  constexpr int kWdTeams = TEAMS;
  constexpr int kWdThreads = TEAMS * kWdWarps * 32;
  typedef typename W::U U;
  constexpr int MA = W::MA, MU = W::MU, KA = W::KA, RA = W::RA, NV = W::NV, PAIR = W::PAIR;
  constexpr bool PH = W::PH, INIT = W::INIT;
  static_assert(SK == SK_M || SK == SK_F || SK == SK_P, "warp-decoupled sweeps: P, M, F");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const unsigned smem_off = (1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + smem_off;

  const int n = P.n, q0 = P.q0, qU = q0 - PAIR;
  const int nst = P.nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * kWdStageBytes);  // nst * teams <= 16
  unsigned char* sp = smem + (size_t)nst * kWdStageBytes + 128;
  double *Jm = nullptr, *Jx = nullptr;
  if (PH) {
    Jm = reinterpret_cast<double*>(sp);
    Jx = Jm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  double* thr = reinterpret_cast<double*>(sp);                          // [RA+1][kWdTT]
  void* PRR = reinterpret_cast<void*>(thr + (kWdRAmax + 1) * kWdTT);  // NV phasors
  double* wsc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(PRR) + 16 * 64);  // per team
  int* blk = reinterpret_cast<int*>(wsc + kWdTeams * 20);  // the block (non-tile) bits
  LRQ_CHECK_SMEM(smem_raw, blk + 64);
  LRQ_CHECK(nst * kWdTeams <= 16 && n <= 40 && q0 + KA - MA <= n);
  int nb = 0;
  for (int j = 0; j < n; ++j)
    if (j >= MA && !(j >= q0 && j < q0 + KA - MA)) ++nb;

  const int bl = qU - MU;  // block unit bits below the high run
  if (threadIdx.x == 0) {
    // full[stage][team]: each barrier has one consumer team that waits on it
    // in order, so its parity (k / (nst * teams)) & 1 is never ambiguous
    for (int s = 0; s < nst; ++s)
      for (int t = 0; t < kWdTeams; ++t) mbar_init(&full[s * kWdTeams + t], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (PH) {
    for (int i = threadIdx.x; i < n * n; i += kWdThreads) Jm[i] = P.J.M[i];
    for (int i = threadIdx.x; i < n; i += kWdThreads) Jx[i] = P.J.ext[i];
    if (threadIdx.x == 0)
      for (int j = 0, m = 0; j < n; ++j)
        if (j >= MA && !(j >= q0 && j < q0 + KA - MA)) blk[m++] = j;
  }
  __syncthreads();
  if (PH) {
    // per tile-thread constants of the phase layout (L2): T_a (a < RA), E_TT
    for (int tt = threadIdx.x; tt < kWdTT; tt += kWdThreads) {
      for (int a = 0; a < RA; ++a) {
        const int ga = W::gpos(W::reg_bit(2, a), q0);
        double acc = 0.0;
        for (int j = 0; j < 7; ++j) {
          const double w = Jm[ga * n + W::gpos(W::thr_bit(2, j), q0)];
          acc += ((tt >> j) & 1) ? -w : w;
        }
        thr[a * kWdTT + tt] = acc;
      }
      double ett = 0.0;
      for (int j = 0; j < 7; ++j) {
        const int gj = W::gpos(W::thr_bit(2, j), q0);
        const double sj = ((tt >> j) & 1) ? -1.0 : 1.0;
        for (int j2 = j + 1; j2 < 7; ++j2) {
          const double w = Jm[gj * n + W::gpos(W::thr_bit(2, j2), q0)];
          ett += (((tt >> j2) & 1) ? -sj : sj) * w;
        }
      }
      thr[RA * kWdTT + tt] = ett;
    }
    for (int v = threadIdx.x; v < NV; v += kWdThreads) {
      double acc = 0.0;
      for (int a = 0; a < RA; ++a) {
        const int ga = W::gpos(W::reg_bit(2, a), q0);
        const double sa = ((v >> a) & 1) ? -1.0 : 1.0;
        for (int b = a + 1; b < RA; ++b) {
          const double w = Jm[ga * n + W::gpos(W::reg_bit(2, b), q0)];
          acc += (((v >> b) & 1) ? -sa : sa) * w;
        }
      }
      if (PAIR) reinterpret_cast<float2*>(PRR)[v] = phasor32(acc);
      else reinterpret_cast<double2*>(PRR)[v] = expmi(acc);
    }
  }
  __syncthreads();
  // The per-tile fields only need the couplings of the block bits: compact
  // tables over the Jm region (they are smaller), so that every warp of a
  // team computes a share of them per tile with independent loads
  //   rowA[m][i] = J[g_i][blk_m] (i < 16), Jb[j][m] = J[blk_j][blk_m],
  //   Jxb[j] = ext[blk_j], gJx[i] = ext[g_i]
  // (complex128 P keeps the direct form below: the tables' extra pointers
  // spill at its 168 registers, +3 % measured)
  constexpr bool TABLES = PH && !(INIT && !PAIR);
  double *rowA = Jm, *Jb = nullptr, *Jxb = nullptr, *gJx = nullptr;
  if (TABLES) {
    Jb = rowA + nb * 16;
    Jxb = Jb + nb * nb;
    gJx = Jxb + nb;
    const int total = nb * 16 + nb * nb + nb + 16;
    constexpr int kMaxPer = 8;
    LRQ_CHECK(total <= kMaxPer * kWdThreads && total <= n * n + n);
    double vals[kMaxPer];
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r) {
      const int e = threadIdx.x + r * kWdThreads;
      double v = 0.0;
      if (e < nb * 16) {
        const int m = e >> 4, i = e & 15;
        v = i < KA ? Jm[W::gpos(i, q0) * n + blk[m]] : 0.0;
      } else if (e < nb * 16 + nb * nb) {
        const int e2 = e - nb * 16, j = e2 / nb, m = e2 - j * nb;
        v = Jm[blk[j] * n + blk[m]];
      } else if (e < nb * 16 + nb * nb + nb) {
        v = Jx[blk[e - nb * 16 - nb * nb]];
      } else if (e < total) {
        const int i = e - nb * 16 - nb * nb - nb;
        v = i < KA ? Jx[W::gpos(i, q0)] : 0.0;
      }
      vals[r] = v;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kMaxPer; ++r) {
      const int e = threadIdx.x + r * kWdThreads;
      if (e < total) rowA[e] = vals[r];
    }
  }
  __syncthreads();

  // refill: the thread that stores a tile loads the tile nst steps ahead
  // into its stage (no producer warp: 8 warps keep 255 registers).  P loads
  // nothing: the same barrier then only says "stage free".
  auto feed = [&](int s, long long k) {
    const long long tid = blockIdx.x + k * (long long)gridDim.x;
    if (tid >= P.num_tiles) return;
    uint64_t* fb = &full[s * kWdTeams + (int)(k % kWdTeams)];
    if constexpr (INIT) {
      mbar_arrive(fb);
    } else {
      void* dst = stages + (size_t)s * kWdStageBytes;
      mbar_expect_tx(fb, kStageBytes);
      const int c1 = (int)((uint64_t)tid & ((1ull << bl) - 1ull)), c4 = (int)((uint64_t)tid >> bl);
      tma_load_5d(dst, &P.tmap, fb, 0, 0, c1, 0, c4);
      // the next tile this CTA will load (fed by the other team about half a
      // tile later) starts its trip to L2 now: that load then hits L2.
      // ($LRQ_WD_PREFETCH = distance in tiles; 1 measured best, 2-4 slower:
      // complex128 F 55.5 / 56.4 / 57.3 / 63.7 ms at n=33)
      if (P.wd_prefetch) {
        const long long nx = tid + (long long)P.wd_prefetch * gridDim.x;
        if (nx < P.num_tiles)
          tma_prefetch_5d(&P.tmap, 0, 0, (int)((uint64_t)nx & ((1ull << bl) - 1ull)), 0, (int)((uint64_t)nx >> bl));
      }
    }
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < nst; ++s) feed(s, s);

  const int team = warp / kWdWarps, wq = warp % kWdWarps;
  const int tt2 = wq | (lane << 2);  // tile-thread index in the phase layout (L2)
  double* hb = wsc + team * 20;      // team: hb[0..KA-1] fields, hb[16..19] warp partials of the block energy
  U r[32];
  constexpr int RPH = INIT ? 0 : 1;  // round of the phase / L2 layout
  const double2 scale = make_double2(P.scale_re, P.scale_im);

  for (long long k = team;; k += kWdTeams) {
    const long long tid = blockIdx.x + k * (long long)gridDim.x;
    if (tid >= P.num_tiles) break;
    const int s = (int)(k % nst);
    U* st = reinterpret_cast<U*>(stages + (size_t)s * kWdStageBytes);
    U* rg = st + wq * kWdRegion;  // this warp's transpose region (after the team barrier)
    const uint64_t ut = (uint64_t)tid;
#ifdef LRQ_CHECKED
    const uint64_t baseU = ((ut & ((1ull << bl) - 1ull)) << MU) | ((ut >> bl) << (qU + kUnitBits - MU));
    LRQ_CHECK((baseU << PAIR) < (1ull << n));
#endif

    if constexpr (PH) {
      // per-tile fields on the tile bits from the block bits, and the block
      // bits' own energy (read after the team barrier below); bit m of the
      // tile index is block bit blk[m].  Complex64 P (no loads: the fields
      // are on the critical path) shares them among the team's 4 warps:
      // fields i = 4 wq + lane / 8 with the block bits split mod 8 over 8
      // lanes, the energy's pairs j < m split mod 4 by warp.  The others leave
      // them to warp 0: the other team's warps issue while this team waits at
      // its barrier, and spreading the work measured slower there
      // (profiles/r02_ab_tile_fields.txt).
      if constexpr (INIT && PAIR) {
        const int i = 4 * wq + (lane >> 3), mm = lane & 7;
        double a = 0.0;
        for (int m = mm; m < nb; m += 8) a = fma(rowA[m * 16 + (i & 15)], spin(ut, m), a);
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        if (mm == 0 && i < KA) hb[i] = gJx[i] + a;
        double tq = 0.0;
        for (int j = lane; j < nb; j += 32) {
          double q = wq == 0 ? Jxb[j] : 0.0;
          for (int m = j + 1 + wq; m < nb; m += kWdWarps) q = fma(Jb[j * nb + m], spin(ut, m), q);
          tq = fma(spin(ut, j), q, tq);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tq += __shfl_xor_sync(0xffffffffu, tq, o);
        if (lane == 0) hb[16 + wq] = tq;
      } else if (!TABLES) {
        if (wq == 0) {
          const uint64_t base = ((ut & ((1ull << bl) - 1ull)) << (MU + PAIR)) |
                                ((ut >> bl) << (qU + kUnitBits - MU + PAIR));
          if (lane < KA) {
            const int gi = W::gpos(lane, q0);
            double acc = Jx[gi];
            for (int m = 0; m < nb; ++m) acc = fma(Jm[gi * n + blk[m]], spin(base, blk[m]), acc);
            hb[lane] = acc;
          }
          double term = 0.0;
          for (int m = lane; m < nb; m += 32) {
            const int j = blk[m];
            double fj = 0.0;
            for (int m2 = 0; m2 < nb; ++m2) fj = fma(Jm[j * n + blk[m2]], spin(base, blk[m2]), fj);
            term += spin(base, j) * (Jx[j] + 0.5 * fj);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
          if (lane < 4) hb[16 + lane] = lane == 0 ? term : 0.0;
        }
      } else if (wq == 0) {
        if (lane < KA) {
          double a = gJx[lane];
          for (int m = 0; m < nb; ++m) a = fma(rowA[m * 16 + lane], spin(ut, m), a);
          hb[lane] = a;
        }
        double tq = 0.0;
        for (int j = lane; j < nb; j += 32) {
          double q = Jxb[j];
          for (int m = j + 1; m < nb; ++m) q = fma(Jb[j * nb + m], spin(ut, m), q);
          tq = fma(spin(ut, j), q, tq);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tq += __shfl_xor_sync(0xffffffffu, tq, o);
        if (lane < 4) hb[16 + lane] = lane == 0 ? tq : 0.0;
      }
    }

    // the k-th tile is the (k / lcm(nst, teams))-th use of its (stage, team) barrier
    mbar_wait(&full[s * kWdTeams + team], (unsigned)((k / (nst % kWdTeams == 0 ? nst : nst * kWdTeams)) & 1));
    if constexpr (!INIT) {
      // L1: lane = unit bits 2..6, registers = unit bits 7..11 (TMA layout)
#pragma unroll
      for (int b = 0; b < 32; ++b) r[b] = st[W::nat(wq, lane, b)];
      if (!PH && !(scale.x == 1.0 && scale.y == 0.0)) W::scale_all(r, scale);
      W::template mix<31u>(r, P.tf[0][0], P.td[0][0]);
      // the 4 warps of the tile have read the TMA layout: the stage is now
      // split into per-warp transpose regions
      team_sync_n(1 + team, kWdWarps * 32);
#pragma unroll
      for (int b = 0; b < 32; ++b) rg[W::slot(lane, b)] = r[b];
      __syncwarp();
      // L2: lane = unit bits 7..11, registers = unit bits 2..6
#pragma unroll
      for (int a = 0; a < 32; ++a) r[a] = rg[W::slot(a, lane)];
      W::template mix<W::L2MASK>(r, P.tf[0][1], P.td[0][1]);
    } else {
      team_sync_n(1 + team, kWdWarps * 32);  // the tile fields are visible
    }

    if constexpr (PH) {
      // phase in L2: E = C + sum_a s_a F_a + E_RR(v)
      double C = (P.J.cst + ((hb[16] + hb[17]) + (hb[18] + hb[19]))) + thr[RA * kWdTT + tt2];
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        const double h = hb[W::thr_bit(2, j)];
        C += ((tt2 >> j) & 1) ? -h : h;
      }
      double F[RA];
#pragma unroll
      for (int a = 0; a < RA; ++a) F[a] = hb[W::reg_bit(2, a)] + thr[a * kWdTT + tt2];
      const double2 sc = INIT ? cmul(scale, make_double2(P.init_re, P.init_im)) : scale;
      W::phase(r, C, F, sc, PRR);
      W::template mix<W::L2MASK>(r, P.tf[1][RPH], P.td[1][RPH]);
    }
    // back to L1 (conflict-free against the TMA layout) through the region
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 32; ++a) rg[W::slot(a, lane)] = r[a];
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 32; ++b) r[b] = rg[W::slot(lane, b)];
    if constexpr (PH) W::template mix<31u>(r, P.tf[1][RPH + 1], P.td[1][RPH + 1]);
    // every warp of the tile is past its region reads: write the tile back in
    // the TMA layout and store it with one bulk tensor copy; the storing
    // thread then refills the stage with the tile nst steps ahead
    team_sync_n(1 + team, kWdWarps * 32);
#pragma unroll
    for (int b = 0; b < 32; ++b) st[W::nat(wq, lane, b)] = r[b];
    fence_proxy_async();
    team_sync_n(1 + team, kWdWarps * 32);
    if (wq == kWdWarps - 1 && lane == 0) {  // the last warp stores
      const int c1 = (int)((uint64_t)tid & ((1ull << bl) - 1ull)), c4 = (int)((uint64_t)tid >> bl);
      tma_store_5d(&P.tmap, st, 0, 0, c1, 0, c4);
      bulk_commit();
      bulk_wait_read<0>();
      feed(s, k + nst);
    }
  }
  if (lane == 0) bulk_wait<0>();  // stores complete before the kernel ends
}

}  // namespace lrq
