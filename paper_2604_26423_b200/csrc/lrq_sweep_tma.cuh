// TMA-fed sweep kernel: one persistent CTA per SM made of TEAMS teams of 8
// warps.  Whole tiles (64 KB, one TMA tensor load each: a 3-D box for a
// contiguous A tile, a 5-D box for the 2^(KA-MA) strided runs of an H tile)
// stream into a ring of NST shared-memory stages; the CTA's k-th tile goes to
// stage k % NST and to team k % TEAMS.  A team runs the same compile-time
// round program as sweep_kernel (lrq_sweep_kernel.cuh), transposing in place
// inside its stage, and stores the result straight from registers.  As soon
// as all 256 threads of the team are past their last shared-memory read of
// the stage, the team's thread 0 refills it with the tile NST steps ahead, so
// loads stay in flight while tiles are computed, and TMA requests are not
// bounded by the LSU miss queue that limits 64/128 B-run register loads.
//
// Stage layout: TMA 128B swizzle (16-byte unit e at e ^ ((e >> 3) & 7)), or
// the 64B swizzle (e ^ ((e >> 3) & 3)) for the 64 B runs of a complex64 H
// tile; every register layout reads it conflict-free except lo = 0 / lo = 2
// (2-way).
#pragma once
#include "lrq_sweep_kernel.cuh"

namespace lrq {

constexpr int kStageBytes = 16 << kUnitBits;  // 64 KB

__host__ __device__ inline size_t tma_smem_bytes(int n, int nst, int teams, bool usesJ, bool usesW) {
  size_t b = (size_t)nst * kStageBytes + 64;  // stages + 3 mbarriers
  if (usesJ) b = align16(b + 8 * (size_t)(n * n + n));
  if (usesW) b = align16(b + 8 * (size_t)(n * n + n));
  b += 8 * (size_t)(((usesJ ? 1 : 0) + (usesW ? 1 : 0)) * 6 * kThreads);  // per-thread constants (shared by teams)
  b = align16(b);
  b += 16 * 32 + 8 * 32 + 8 * 32;                                    // PRR, PRR32, ERR
  b += (size_t)teams * 8 * (2 * 2 * 16 + 4 + 5 * (kThreads / 32));  // per team: hB, EBB, reduce scratch
  return align16(b) + 1024;  // slack for the 1024-byte stage alignment
}

// the load ring of one CTA
struct Feed {
  const CUtensorMap* tmap;
  unsigned char* stages;
  uint64_t* full;  // [stage][team] (6 barriers)
  int nst, bl, teams;
  long long num_tiles;
};

// The load of the CTA's k-th tile completes on full[s][k % teams]: each
// (stage, team) barrier then completes in exactly the order its one consumer
// team waits on it, so parity (k / lcm(nst, teams)) & 1 is never ambiguous
// (one barrier per stage shared by two teams would let a team that ran ahead
// observe the previous phase).
__device__ __forceinline__ uint64_t* full_bar(const Feed& f, int s, long long k) {
  return &f.full[s * 2 + (int)(k % f.teams)];
}

template <int GK>
__device__ __forceinline__ void feed_tile(const Feed& f, int s, long long k, long long tid) {
  void* dst = f.stages + (size_t)s * kStageBytes;
  uint64_t* bar = full_bar(f, s, k);
  mbar_expect_tx(bar, kStageBytes);
  if constexpr (GK == GK_A) {
    tma_load_3d(dst, f.tmap, bar, 0, 0, (int)(2 * tid));
  } else {
    const int c1 = (int)((uint64_t)tid & ((1ull << f.bl) - 1ull)), c4 = (int)((uint64_t)tid >> f.bl);
    tma_load_5d(dst, f.tmap, bar, 0, 0, c1, 0, c4);
  }
}

template <typename T, int GK, int SK>
struct TmaSweep {
  typedef SweepCtx<T, GK, SK> S;
  typedef SweepTile<T, GK, SK> W;
  typedef typename S::U U;
  typedef typename W::Ctx Ctx;
  static constexpr int PAIR = S::PAIR, NR = S::NR;

  // TMA swizzle of the stage: 128B rows (mask 7); the 64 B runs of a complex64
  // H tile use the 64B mode (mask 3) so the box is not padded to 128 B rows
  static constexpr int SWM = (GK == GK_H && PAIR) ? 3 : 7;
  __device__ static __forceinline__ int swz(int e) { return e ^ ((e >> 3) & SWM); }

  template <int LO>
  __device__ static __forceinline__ void to_smem(U* st, const U (&r)[16], int t) {
    const int eb = S::ebase(t, LO);
#pragma unroll
    for (int j = 0; j < 16; ++j) st[swz(eb | (j << LO))] = r[j];
  }
  template <int LO>
  __device__ static __forceinline__ void from_smem(const U* st, U (&r)[16], int t) {
    const int eb = S::ebase(t, LO);
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = st[swz(eb | (j << LO))];
  }

  // last round whose start reads the stage (0: only the initial load)
  __host__ __device__ static constexpr int last_smem_round() {
    int last = 0;
    for (int r = 1; r < NR; ++r)
      if (prog_lo(GK, PAIR, SK, r) != prog_lo(GK, PAIR, SK, r - 1)) last = r;
    return last;
  }

  // every thread of the team is past its last access of stage s: refill it
  // with the CTA's tile nst steps ahead (generic-proxy accesses fenced first)
  __device__ static __forceinline__ void release(const Feed& f, int s, long long k, const Ctx& c) {
    fence_proxy_async();
    team_sync(c.bar);
    const long long nxt = blockIdx.x + (k + f.nst) * (long long)gridDim.x;
    if (c.t == 0 && nxt < f.num_tiles) feed_tile<GK>(f, s, k + f.nst, nxt);
  }

  template <int RR>
  __device__ static __forceinline__ void round(Ctx& c, const Feed& f, int s, long long k) {
    constexpr int LO = prog_lo(GK, PAIR, SK, RR);
    if constexpr (RR > 0) {
      constexpr int PREV = prog_lo(GK, PAIR, SK, RR - 1);
      if constexpr (LO != PREV) {
        team_sync(c.bar);  // every thread is done reading the old layout
        to_smem<PREV>(c.tile, c.r, c.t);
        team_sync(c.bar);
        from_smem<LO>(c.tile, c.r, c.t);
        if constexpr (RR == last_smem_round()) release(f, s, k, c);
      }
    }
    constexpr unsigned M1 = prog_mask(GK, PAIR, SK, RR, 0);
    constexpr unsigned M2 = prog_mask(GK, PAIR, SK, RR, 1);
    if constexpr (M1 != 0) S::template mix<M1>(c.r, c.P->tf[0][RR], c.P->td[0][RR]);
    if constexpr (prog_phase(SK, GK, PAIR, RR)) W::phase(c, LO);
    if constexpr (M2 != 0) S::template mix<M2>(c.r, c.P->tf[1][RR], c.P->td[1][RR]);
    if constexpr (prog_reduce(SK, GK, PAIR, RR)) {
      if (SK != SK_L || c.P->reduce) W::reduce(c, LO);
    }
  }

  template <int... RR>
  __device__ static __forceinline__ void rounds(Ctx& c, const Feed& f, int s, long long k,
                                                std::integer_sequence<int, RR...>) {
    (round<RR>(c, f, s, k), ...);
  }
};

template <typename T, int GK, int SK, int TEAMS>
__global__ void __launch_bounds__(TEAMS* kThreads, 1) sweep_tma_kernel(const __grid_constant__ SweepParams P) {
  typedef SweepCtx<T, GK, SK> S;
  typedef SweepTile<T, GK, SK> W;
  typedef TmaSweep<T, GK, SK> X;
  typedef typename S::U U;
  typedef typename S::A A;
  constexpr int PAIR = S::PAIR, NV = S::NV, NR = S::NR, MU = S::MU;
  constexpr bool HAS_PHASE = SK == SK_F || SK == SK_L;
  constexpr bool HAS_REDUCE = SK == SK_R || SK == SK_L || SK == SK_Q;
  static_assert(SK != SK_P && SK != SK_N, "the TMA path serves sweeps that load the state");
  constexpr int LO_PHASE = HAS_PHASE ? prog_lo(GK, PAIR, SK, SK == SK_F ? num_layouts(GK, PAIR) - 1 : 0) : 0;
  constexpr int LO_RED = prog_lo(GK, PAIR, SK, NR - 1);
  extern __shared__ __align__(1024) unsigned char smem_raw[];

  const int n = P.n, q0 = P.q0, qU = q0 - PAIR;
  const int team = threadIdx.x / kThreads;
  const int t = threadIdx.x % kThreads;
  const int nst = P.nstages;
  const bool usesW = HAS_REDUCE && (SK != SK_L || P.reduce);

  // 1024-byte alignment for the swizzled TMA stages, as an offset into the
  // __shared__ array: a pointer laundered through uintptr_t would lose the
  // address space and turn every stage / table access into a generic LD/ST
  const unsigned smem_off = (1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + smem_off;
  unsigned char* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * kStageBytes);
  unsigned char* sp = smem + (size_t)nst * kStageBytes + 64;
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
  double* thr = reinterpret_cast<double*>(sp);           // phase matrix constants
  double* thrW = thr + (HAS_PHASE ? 6 * kThreads : 0);  // cost matrix constants
  sp = smem + align16((size_t)(reinterpret_cast<unsigned char*>(thrW + (usesW ? 6 * kThreads : 0)) - smem));
  double2* PRR = reinterpret_cast<double2*>(sp);
  float2* PRR32 = reinterpret_cast<float2*>(PRR + 32);
  double* ERR = reinterpret_cast<double*>(PRR32 + 32);
  double* teamb = ERR + 32 + team * (2 * 2 * 16 + 4 + 5 * (kThreads / 32));
  double* hB = teamb;
  double* EBB = hB + 2 * 2 * 16;
  double* rs = EBB + 4;

  const int bl = qU - MU;
  Feed f;
  f.tmap = &P.tmap;
  f.stages = stages;
  f.full = full;
  f.nst = nst;
  f.teams = TEAMS;
  f.bl = bl;
  f.num_tiles = P.num_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 6; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < nst; ++s) {  // prologue: the CTA's first nst tiles
      const long long tid = blockIdx.x + (long long)s * gridDim.x;
      if (tid < P.num_tiles) feed_tile<GK>(f, s, s, tid);
    }
  }
  for (int i = threadIdx.x; i < n * n; i += TEAMS * kThreads) {
    if (HAS_PHASE) Jm[i] = P.J.M[i];
    if (usesW) Wm[i] = P.W.M[i];
  }
  for (int i = threadIdx.x; i < n; i += TEAMS * kThreads) {
    if (HAS_PHASE) Jx[i] = P.J.ext[i];
    if (usesW) Wx[i] = P.W.ext[i];
  }
  __syncthreads();
  if (team == 0) {
    if (HAS_PHASE) {
      S::thread_consts(Jm, n, q0, LO_PHASE, t, thr);
      if (t < NV) {
        const double e = S::err_entry(Jm, n, q0, LO_PHASE, t);
        PRR[t] = expmi(e);
        PRR32[t] = phasor32(e);
      }
    }
    if (usesW) {
      S::thread_consts(Wm, n, q0, LO_RED, t, thrW);
      if (t < NV) ERR[t] = S::err_entry(Wm, n, q0, LO_RED, t);
    }
  }
  __syncthreads();

  typename W::Ctx c;
  c.P = &P;
  c.thr = thr;
  c.thrW = thrW;
  c.PRR = PRR;
  c.PRR32 = PRR32;
  c.ERR = ERR;
  c.rs = rs;
  c.shist = nullptr;  // the histogram runs on the register path (launch_sweep)
  c.t = t;
  c.q0 = q0;
  c.qU = qU;
  c.bar = 1 + team;
  U* gamps = reinterpret_cast<U*>(P.amps);

  int par = 0;
  for (long long k = team;; k += TEAMS, par ^= 1) {
    const long long tid = blockIdx.x + k * (long long)gridDim.x;
    if (tid >= P.num_tiles) break;
    const int s = (int)(k % nst);
    U* st = reinterpret_cast<U*>(stages + (size_t)s * kStageBytes);
    const uint64_t ut = (uint64_t)tid;
    const uint64_t baseU = ((ut & ((1ull << bl) - 1ull)) << MU) | ((ut >> bl) << (qU + kUnitBits - MU));
    c.base = baseU << PAIR;
    c.tid = tid;
    c.tile = st;
    double* hbJ = hB + (par * 2 + 0) * 16;
    double* hbW = hB + (par * 2 + 1) * 16;
    if (HAS_PHASE) S::block_consts(Jm, Jx, P.J.cst, n, q0, c.base, 0, hbJ, &EBB[par * 2 + 0], t);
    if (usesW) S::block_consts(Wm, Wx, P.W.cst, n, q0, c.base, 2, hbW, &EBB[par * 2 + 1], t);
    team_sync(c.bar);
    c.hbJ = hbJ;
    c.hbW = hbW;
    c.ebbJ = EBB[par * 2 + 0];
    c.ebbW = EBB[par * 2 + 1];

    mbar_wait(full_bar(f, s, k), (unsigned)((k / (nst == TEAMS ? nst : nst * TEAMS)) & 1));
    X::template from_smem<prog_lo(GK, PAIR, SK, 0)>(st, c.r, t);
    if constexpr (X::last_smem_round() == 0) X::release(f, s, k, c);
    if (!HAS_PHASE && !(P.scale_re == 1.0 && P.scale_im == 0.0)) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        A x = amp_get(c.r, v);
        if (P.scale_im == 0.0) {
          x.x *= (T)P.scale_re;
          x.y *= (T)P.scale_re;
        } else {
          x = cmul_amp(x, make_double2(P.scale_re, P.scale_im));
        }
        amp_set(c.r, v, x);
      }
    }

    X::rounds(c, f, s, k, std::make_integer_sequence<int, NR>{});

    if constexpr (SK != SK_Q) {
      constexpr int LO = prog_store_lo(GK, PAIR, SK);
      const int eb = S::ebase(t, LO);
      U* g = gamps + baseU + S::gunit(eb, qU);
      const int sh = S::gshift(LO, qU);
#pragma unroll
      for (int j = 0; j < 16; ++j) st_unit(g + ((uint64_t)j << sh), c.r[j]);
    }
  }
}

}  // namespace lrq
