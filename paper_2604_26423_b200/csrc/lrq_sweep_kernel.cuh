// sweep_kernel: persistent CTAs (2 per SM) walk the tiles of one sweep; per
// tile the compile-time round program of (GK, SK) runs fully unrolled, so
// every shared-memory address is base + immediate and every butterfly is
// straight-line FP code (see lrq_sweep.cuh for the programs and layouts).
#pragma once
#include <utility>

#include "lrq_sweep.cuh"

namespace lrq {

template <typename T, int GK, int SK>
struct SweepTile {
  typedef SweepCtx<T, GK, SK> S;
  typedef typename S::U U;
  typedef typename S::A A;
  static constexpr int PAIR = S::PAIR, RA = S::RA, NV = S::NV, NR = S::NR;
  static constexpr bool INIT = SK == SK_P;
  static constexpr bool AMPS = SK != SK_N;

  // everything a round needs, per thread and per tile
  struct Ctx {
    U r[16];
    const SweepParams* P;
    U* tile;
    const double* thr;   // per-thread constants of the phase matrix [6][kThreads]
    const double* thrW;  // per-thread constants of the cost matrix [6][kThreads]
    const double* hbJ;  // per-tile fields (phase matrix)
    const double* hbW;  // per-tile fields (cost matrix)
    double ebbJ, ebbW;
    const double2* PRR;
    const float2* PRR32;
    const double* ERR;
    double* rs;
    unsigned long long* shist;  // shared energy histogram (null: off)
    uint64_t base;  // amp index of tile element 0
    long long tid;
    int t, q0, qU;
    int bar;  // named barrier of this 256-thread team
  };

  // complex64: the angles are assembled and reduced mod 2pi in float64, the
  // unit phasors and their products are float32 (error ~1e-6, far inside the
  // 1e-5 complex64 tolerance and below the reference's own fp32 drift)
  __device__ static __forceinline__ void phase(Ctx& c, int lo) {
    // E_J(v) = C + sum_a s_a F_a + E_RR(v); exp(-i E_J) in product form
    const double* th = c.thr;
    double F[RA];
    double C = c.ebbJ + th[RA * kThreads + c.t];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double h = c.hbJ[thr_tile_bit(PAIR, lo, j)];
      C += ((c.t >> j) & 1) ? -h : h;
    }
#pragma unroll
    for (int a = 0; a < RA; ++a) F[a] = c.hbJ[reg_tile_bit(PAIR, lo, a)] + th[a * kThreads + c.t];
    if constexpr (PAIR) {
      const double2 sc = make_double2(c.P->scale_re, c.P->scale_im);
      double2 s2 = sc;
      if constexpr (INIT) s2 = cmul(sc, make_double2(c.P->init_re, c.P->init_im));
      const float2 eC = cmul32(make_float2((float)s2.x, (float)s2.y), phasor32(C));
      const float2 u0 = phasor32(F[0]), u1 = phasor32(F[1]), u2 = phasor32(F[2]), u3 = phasor32(F[3]),
                   u4 = phasor32(F[4]);
      const float2 p01 = cmul32(u0, u1), q01 = cmul32_conj(u1, u0);
      float2 Alo[4];
      Alo[0] = cmul32(eC, p01);
      Alo[1] = cmul32(eC, q01);
      Alo[2] = cmul32_conj(eC, q01);
      Alo[3] = cmul32_conj(eC, p01);
      const float2 p23 = cmul32(u2, u3), q23 = cmul32_conj(u3, u2);
      const float2 Y[4] = {p23, q23, conj32(q23), conj32(p23)};
      const float2* PRR32 = c.PRR32;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const float2 Bh = (h & 4) ? cmul32_conj(Y[h & 3], u4) : cmul32(Y[h & 3], u4);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const int v = h * 4 + l;
          const float2 ph = cmul32(cmul32(Alo[l], Bh), PRR32[v]);
          if constexpr (INIT) amp_set(c.r, v, ph);
          else amp_set(c.r, v, cmul32(amp_get(c.r, v), ph));
        }
      }
      return;
    }
    double2 eC = cmul(make_double2(c.P->scale_re, c.P->scale_im), expmi(C));
    if constexpr (INIT) eC = cmul(eC, make_double2(c.P->init_re, c.P->init_im));
    const double2 u0 = expmi(F[0]), u1 = expmi(F[1]), u2 = expmi(F[2]), u3 = expmi(F[3]);
    const double2 p01 = cmul(u0, u1), q01 = cmul_conj(u1, u0);  // u0 u1, conj(u0) u1
    double2 Alo[4];
    Alo[0] = cmul(eC, p01);
    Alo[1] = cmul(eC, q01);
    Alo[2] = cmul_conj(eC, q01);  // eC u0 conj(u1)
    Alo[3] = cmul_conj(eC, p01);
    const double2 p23 = cmul(u2, u3), q23 = cmul_conj(u3, u2);
    double2 Y[4];
    Y[0] = p23;
    Y[1] = q23;
    Y[2] = make_double2(q23.x, -q23.y);
    Y[3] = make_double2(p23.x, -p23.y);
    double2 u4 = make_double2(1.0, 0.0);
    if constexpr (RA == 5) u4 = expmi(F[4]);
#pragma unroll
    for (int h = 0; h < NV / 4; ++h) {
      double2 Bh = Y[h & 3];
      if constexpr (RA == 5) Bh = (h & 4) ? cmul_conj(Bh, u4) : cmul(Bh, u4);
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const int v = h * 4 + l;
        const double2 ph = cmul(cmul(Alo[l], Bh), c.PRR[v]);
        if constexpr (INIT) {
          A x;
          x.x = (T)ph.x;
          x.y = (T)ph.y;
          amp_set(c.r, v, x);
        } else {
          amp_set(c.r, v, cmul_amp(amp_get(c.r, v), ph));
        }
      }
    }
  }

  template <bool SEARCH, bool HIST>
  __device__ static __forceinline__ void reduce_loop(Ctx& c, const SweepParams& P, const double (&Elo)[4],
                                                     const double (&Fh)[3], unsigned vmask, bool thread_ok,
                                                     double& sp_, double& spe, double& mine, double& maxe,
                                                     int& bestv) {
    double eh = 0.0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if ((v & 3) == 0) {
        const int h = v >> 2;
        eh = ((h & 1) ? -Fh[0] : Fh[0]) + ((h & 2) ? -Fh[1] : Fh[1]);
        if constexpr (RA == 5) eh += (h & 4) ? -Fh[2] : Fh[2];
      }
      const double ev = (Elo[v & 3] + eh) + c.ERR[v];
      if constexpr (AMPS) {
        const double pv = prob(amp_get(c.r, v));
        sp_ += pv;
        spe = fma(pv, ev, spe);
        if constexpr (HIST) hist_add(c.shist, P.hist_bins, P.hist_lo, P.hist_scale, ev, pv);
      }
      if constexpr (SEARCH) {
        maxe = fmax(maxe, ev);
        if (thread_ok && !(v & vmask) && ev < mine) {
          mine = ev;
          bestv = v;
        }
      }
    }
  }

  __device__ static __forceinline__ void reduce(Ctx& c, int lo) {
    const SweepParams& P = *c.P;
    const double* th = c.thrW;
    double F[RA];
    double C = c.ebbW + th[RA * kThreads + c.t];
    bool thread_ok = true;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = thr_tile_bit(PAIR, lo, j);
      const double h = c.hbW[i];
      const bool bit = (c.t >> j) & 1;
      C += bit ? -h : h;
      if (bit && S::gpos(i, c.q0) == P.min_bit) thread_ok = false;
    }
    unsigned vmask = 0;
#pragma unroll
    for (int a = 0; a < RA; ++a) {
      const int i = reg_tile_bit(PAIR, lo, a);
      F[a] = c.hbW[i] + th[a * kThreads + c.t];
      if (S::gpos(i, c.q0) == P.min_bit) vmask = 1u << a;
    }
    if (P.min_bit == -2 || (P.min_bit >= 0 && ((c.base >> P.min_bit) & 1ull))) thread_ok = false;
    // E(v) = (Elo[v & 3] + Ehi(v >> 2)) + ERR[v]; Ehi is formed inside the
    // loop (fewer live registers: the R kernel runs 2 CTAs per SM)
    double Elo[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) Elo[l] = C + ((l & 1) ? -F[0] : F[0]) + ((l & 2) ? -F[1] : F[1]);
    const double Fh[3] = {F[2], F[3], RA == 5 ? F[4] : 0.0};
    double sp_ = 0.0, spe = 0.0, mine = __longlong_as_double(0x7ff0000000000000ll);
    double maxe = -__longlong_as_double(0x7ff0000000000000ll);
    int bestv = NV;
    // the per-amplitude loop in three compile-time forms: plain sums (the
    // max-cut optimum already known), + min/argmin/max E search, + histogram
    if (!AMPS || P.search) {
      if (AMPS && c.shist)
        reduce_loop<true, true>(c, P, Elo, Fh, vmask, thread_ok, sp_, spe, mine, maxe, bestv);
      else
        reduce_loop<true, false>(c, P, Elo, Fh, vmask, thread_ok, sp_, spe, mine, maxe, bestv);
    } else {
      if (c.shist)
        reduce_loop<false, true>(c, P, Elo, Fh, vmask, thread_ok, sp_, spe, mine, maxe, bestv);
      else
        reduce_loop<false, false>(c, P, Elo, Fh, vmask, thread_ok, sp_, spe, mine, maxe, bestv);
    }
    unsigned long long zbest = ~0ull;
    if (bestv < NV) {
      const int eU = S::ebase(c.t, lo) | ((bestv >> PAIR) << lo);
      zbest = c.base + (S::gunit(eU, c.qU) << PAIR) + (uint64_t)(bestv & PAIR);
    }
    // without the search the extremes are the constants set above: only the
    // two sums need the warp reduction
    const bool full = !AMPS || P.search;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sp_ += __shfl_xor_sync(0xffffffffu, sp_, o);
      spe += __shfl_xor_sync(0xffffffffu, spe, o);
      if (full) {
        const double om = __shfl_xor_sync(0xffffffffu, mine, o);
        const unsigned long long oz = __shfl_xor_sync(0xffffffffu, zbest, o);
        if (om < mine || (om == mine && oz < zbest)) {
          mine = om;
          zbest = oz;
        }
        maxe = fmax(maxe, __shfl_xor_sync(0xffffffffu, maxe, o));
      }
    }
    const int warp = c.t >> 5;
    if ((c.t & 31) == 0) {
      c.rs[warp * 5 + 0] = sp_;
      c.rs[warp * 5 + 1] = spe;
      c.rs[warp * 5 + 2] = mine;
      c.rs[warp * 5 + 3] = __longlong_as_double((long long)zbest);
      c.rs[warp * 5 + 4] = maxe;
    }
    team_sync(c.bar);  // the 256 threads of this team only
    if (c.t == 0) {
      double s0 = 0.0, s1 = 0.0, mn = c.rs[2], mx = c.rs[4];
      unsigned long long zb = (unsigned long long)__double_as_longlong(c.rs[3]);
      for (int w = 0; w < kThreads / 32; ++w) {
        s0 += c.rs[w * 5 + 0];
        s1 += c.rs[w * 5 + 1];
        if (!full) continue;
        const double om = c.rs[w * 5 + 2];
        const unsigned long long oz = (unsigned long long)__double_as_longlong(c.rs[w * 5 + 3]);
        if (om < mn || (om == mn && oz < zb)) {
          mn = om;
          zb = oz;
        }
        mx = fmax(mx, c.rs[w * 5 + 4]);
      }
      P.red_p[c.tid] = s0;
      P.red_pE[c.tid] = s1;
      P.red_minE[c.tid] = mn;
      P.red_arg[c.tid] = zb;
      if (P.red_maxE) P.red_maxE[c.tid] = mx;
    }
  }

  template <int RR>
  __device__ static __forceinline__ void round(Ctx& c) {
    constexpr int LO = prog_lo(GK, PAIR, SK, RR);
    if constexpr (AMPS && RR > 0) {
      constexpr int PREV = prog_lo(GK, PAIR, SK, RR - 1);
      if constexpr (LO != PREV) {
        if constexpr (RR > 1) __syncthreads();  // the previous layout's reads are done
        S::template to_smem<PREV>(c.tile, c.r, c.t);
        __syncthreads();
        S::template from_smem<LO>(c.tile, c.r, c.t);
      }
    }
    constexpr unsigned M1 = prog_mask(GK, PAIR, SK, RR, 0);
    constexpr unsigned M2 = prog_mask(GK, PAIR, SK, RR, 1);
    if constexpr (M1 != 0) S::template mix<M1>(c.r, c.P->tf[0][RR], c.P->td[0][RR]);
    if constexpr (prog_phase(SK, GK, PAIR, RR)) phase(c, LO);
    if constexpr (M2 != 0) S::template mix<M2>(c.r, c.P->tf[1][RR], c.P->td[1][RR]);
    if constexpr (prog_reduce(SK, GK, PAIR, RR)) {
      if (SK != SK_L || c.P->reduce) reduce(c, LO);
    }
  }

  template <int... RR>
  __device__ static __forceinline__ void rounds(Ctx& c, std::integer_sequence<int, RR...>) {
    (round<RR>(c), ...);
  }
};

template <typename T, int GK, int SK>
__global__ void __launch_bounds__(kThreads, 2) sweep_kernel(const __grid_constant__ SweepParams P) {
  typedef SweepCtx<T, GK, SK> S;
  typedef SweepTile<T, GK, SK> W;
  typedef typename S::U U;
  typedef typename S::A A;
  constexpr int PAIR = S::PAIR, NV = S::NV, NR = S::NR, MU = S::MU;
  constexpr bool INIT = SK == SK_P;
  constexpr bool AMPS = SK != SK_N;
  constexpr bool STORE = SK != SK_Q && SK != SK_N;
  constexpr bool HAS_PHASE = SK == SK_P || SK == SK_F || SK == SK_L;
  constexpr bool HAS_REDUCE = SK == SK_R || SK == SK_L || SK == SK_Q || SK == SK_N;
  constexpr int LO_PHASE = HAS_PHASE ? prog_lo(GK, PAIR, SK, SK == SK_F ? num_layouts(GK, PAIR) - 1 : 0) : 0;
  constexpr int LO_RED = prog_lo(GK, PAIR, SK, NR - 1);
  extern __shared__ __align__(16) unsigned char smem[];

  const int n = P.n, q0 = P.q0, qU = q0 - PAIR;
  const int t = threadIdx.x;
  const bool usesW = HAS_REDUCE && (SK != SK_L || P.reduce);

  unsigned char* sp = smem;
  U* tile = reinterpret_cast<U*>(sp);
  if (AMPS) sp += 16 * (size_t)kTileUnitsPadded;
  double *Jm = nullptr, *Jx = nullptr, *Wm = nullptr, *Wx = nullptr;
  if (HAS_PHASE) {
    Jm = reinterpret_cast<double*>(sp);
    Jx = Jm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  if (usesW) {
    Wm = reinterpret_cast<double*>(sp);
    Wx = Wm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  double* hB = reinterpret_cast<double*>(sp);  // [parity][mat][16]
  double* EBB = hB + 2 * 2 * 16;               // [parity][mat]
  double* thr = EBB + 4;                       // [mat][6][kThreads]
  sp = smem + align16((size_t)(reinterpret_cast<unsigned char*>(thr + 2 * 6 * kThreads) - smem));
  double2* PRR = reinterpret_cast<double2*>(sp);
  float2* PRR32 = reinterpret_cast<float2*>(PRR + 32);
  double* ERR = reinterpret_cast<double*>(PRR32 + 32);
  double* rs = ERR + 32;
  unsigned long long* shist = reinterpret_cast<unsigned long long*>(rs + 5 * (kThreads / 32));
  LRQ_CHECK_SMEM(smem, shist + (HAS_REDUCE && P.hist ? P.hist_bins : 0));
  LRQ_CHECK(P.n <= 40 && q0 >= S::MA && (GK == GK_A || q0 + kUnitBits + PAIR - S::MA <= n));
  const bool hist = HAS_REDUCE && AMPS && P.hist != nullptr;
  if (hist)
    for (int i = t; i < P.hist_bins; i += kThreads) shist[i] = 0ull;

  for (int i = t; i < n * n; i += kThreads) {
    if (HAS_PHASE) Jm[i] = P.J.M[i];
    if (usesW) Wm[i] = P.W.M[i];
  }
  for (int i = t; i < n; i += kThreads) {
    if (HAS_PHASE) Jx[i] = P.J.ext[i];
    if (usesW) Wx[i] = P.W.ext[i];
  }
  __syncthreads();
  if (HAS_PHASE) {
    S::thread_consts(Jm, n, q0, LO_PHASE, t, thr);
    if (t < NV) {
      const double e = S::err_entry(Jm, n, q0, LO_PHASE, t);
      PRR[t] = expmi(e);
      PRR32[t] = phasor32(e);
    }
  }
  if (usesW) {
    S::thread_consts(Wm, n, q0, LO_RED, t, thr + 6 * kThreads);
    if (t < NV) ERR[t] = S::err_entry(Wm, n, q0, LO_RED, t);
  }

  typename W::Ctx c;
  c.P = &P;
  c.tile = tile;
  c.thr = thr;
  c.thrW = thr + 6 * kThreads;
  c.PRR = PRR;
  c.PRR32 = PRR32;
  c.ERR = ERR;
  c.rs = rs;
  c.shist = hist ? shist : nullptr;
  c.t = t;
  c.q0 = q0;
  c.qU = qU;
  c.bar = 1;
  U* gamps = reinterpret_cast<U*>(P.amps);
  const int bl = qU - MU;  // block unit bits below the high run

  // per-launch scalars held in registers across the tile loop (a reload from
  // the parameter bank after every barrier stalled the loop: the parameter
  // block is larger than the constant cache); the empty asm keeps the
  // compiler from re-materialising them as constant loads
  // scale mode: 0 none, 1 real, 2 complex
  int smode = (P.scale_re == 1.0 && P.scale_im == 0.0) ? 0 : (P.scale_im == 0.0 ? 1 : 2);
  float sre32 = (float)P.scale_re;
  unsigned ntile = (unsigned)P.num_tiles;
  asm volatile("" : "+r"(smode), "+f"(sre32), "+r"(ntile));
  int par = 0;
  for (unsigned tid32 = blockIdx.x; tid32 < ntile; tid32 += gridDim.x, par ^= 1) {
    const long long tid = tid32;
    LRQ_CHECK(tid < P.num_tiles);
    const uint64_t ut = (uint64_t)tid;
    const uint64_t baseU = ((ut & ((1ull << bl) - 1ull)) << MU) | ((ut >> bl) << (qU + kUnitBits - MU));
    c.base = baseU << PAIR;
    c.tid = tid;

    if constexpr (AMPS && !INIT) {
      constexpr int LO = prog_lo(GK, PAIR, SK, 0);
      const int eb = S::ebase(t, LO);
      const U* g = gamps + baseU + S::gunit(eb, qU);
      const int sh = S::gshift(LO, qU);
#pragma unroll
      for (int j = 0; j < 16; ++j) c.r[j] = ld_unit(g + ((uint64_t)j << sh));
      // group A: pull this CTA's next (contiguous, 64 KB) tile into L2 with one
      // TMA bulk prefetch while the current one is computed.  (For the strided
      // H tiles the 2^(12-MU) small prefetches cost more than they hide.)
      if (t == 0) {
        const long long nxt = tid + gridDim.x;
        if constexpr (GK == GK_A) {
          if (nxt < P.num_tiles) prefetch_l2(gamps + ((uint64_t)nxt << kUnitBits), 16u << kUnitBits);
        } else {
          // one TMA tensor prefetch covers all 2^(12-MU) strided runs of the tile
          if (P.has_tmap && nxt < P.num_tiles) {
            const int c1 = (int)((uint64_t)nxt & ((1ull << bl) - 1ull)), c4 = (int)((uint64_t)nxt >> bl);
            tma_prefetch_5d(&P.tmap, 0, 0, c1, 0, c4);
          }
        }
      }
    }

    // the tile's block constants (serial fp64 chains on two warps) are
    // computed while its loads are in flight; hB[par] was last read two
    // tiles ago, before the previous tile's barrier
    double* hbJ = hB + (par * 2 + 0) * 16;
    double* hbW = hB + (par * 2 + 1) * 16;
    if (HAS_PHASE) S::block_consts(Jm, Jx, P.J.cst, n, q0, c.base, 0, hbJ, &EBB[par * 2 + 0], t);
    if (usesW) S::block_consts(Wm, Wx, P.W.cst, n, q0, c.base, 2, hbW, &EBB[par * 2 + 1], t);
    __syncthreads();
    c.hbJ = hbJ;
    c.hbW = hbW;
    c.ebbJ = EBB[par * 2 + 0];
    c.ebbW = EBB[par * 2 + 1];
    if constexpr (AMPS && !INIT && !HAS_PHASE) {
      if (smode == 1) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          A x = amp_get(c.r, v);
          if constexpr (PAIR) {
            x.x *= sre32;
            x.y *= sre32;
          } else {
            x.x *= P.scale_re;
            x.y *= P.scale_re;
          }
          amp_set(c.r, v, x);
        }
      } else if (smode == 2) {
#pragma unroll
        for (int v = 0; v < NV; ++v) amp_set(c.r, v, cmul_amp(amp_get(c.r, v), make_double2(P.scale_re, P.scale_im)));
      }
    }

    W::rounds(c, std::make_integer_sequence<int, NR>{});

    if constexpr (STORE) {
      constexpr int LO = prog_store_lo(GK, PAIR, SK);
      const int eb = S::ebase(t, LO);
      U* gbase = gamps + baseU;
      if constexpr (GK == GK_A && SK == SK_M) {
        if (P.remap)  // group-A tiles are contiguous: the whole tile goes to one rank
          gbase = reinterpret_cast<U*>(P.rdst[tid >> P.rbits]) + ((uint64_t)(tid & ((1ll << P.rbits) - 1)) << kUnitBits);
      }
      U* g = gbase + S::gunit(eb, qU);
      const int sh = S::gshift(LO, qU);
#pragma unroll
      for (int j = 0; j < 16; ++j) st_unit(g + ((uint64_t)j << sh), c.r[j]);
    }
  }
  if (hist) {  // the CTA's histogram into the global one (integer adds: any order)
    __syncthreads();
    for (int i = t; i < P.hist_bins; i += kThreads)
      if (shist[i]) atomicAdd(P.hist + i, shist[i]);
  }
}

}  // namespace lrq
