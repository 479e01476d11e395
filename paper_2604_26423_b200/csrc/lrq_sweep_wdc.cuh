// Cluster-pair sweeps of a high qubit group with a 128 KB tile (complex64):
// the P, M and F sweeps of the "C" groups.
//
// Why: a high-group tile is 2^k runs of 2^MA contiguous amplitudes, and the
// DRAM efficiency of a run grows with its length: a compute-free copy of
// 64 B runs at the n=32 strides moves 4.3-4.7 TB/s, 128 B runs 4.6-5.0,
// 256 B runs 5.7-6.0 (profiles/r02_run_copy_n32.txt).  One SM's shared
// memory holds 64 KB tiles (three stages in flight), so a group of k = 10
// targets there has 64 B runs.  Two CTAs of a cluster together hold a
// 128 KB tile: k = 10 targets with 128 B runs (group C10) or 9 with 256 B
// runs (C9), 8 with 512 B (C8).
//
// Each CTA of the pair holds one half of the tile: the halves differ in the
// group's top target qubit c (the "cross" qubit), CTA rank = bit c.  A half
// is laid out exactly like a 64 KB warp-decoupled tile (lrq_sweep_wd.cuh,
// WdSweep) with the k-1 local targets, so the butterflies of the local
// targets, the cost phase (bit c enters as a block bit) and the per-warp
// transposes are the single-CTA code.  Only the cross qubit needs the other
// half.  Mixers of different qubits commute and the phase is diagonal, so
// an F sweep's mix1(c) -> phase -> mix2(c) on the pair (x: this CTA's
// amplitude after the local mix1, y: the partner's at the same position) is
// one fused update per amplitude, with ONE exchange:
//     out = phi_m [ (x + i t1 y) + i t2 K (y + i t1 x) ],   K = phi_p / phi_m
// where phi_m, phi_p are the cost phases of the two amplitudes (they differ
// by the flipped spin s_c: K = exp(2 i s_c h_c), h_c the field on c).  Each
// warp writes its post-mix1 values into its transpose region, the matching
// warp of the partner CTA reads them through distributed shared memory
// (ld.shared::cluster), and two per-warp cluster-scope mbarriers order it:
// "my region is ready" (arrived remotely by the partner's 32 lanes) and
// "the partner has read my region" (before the region is reused).  DSMEM
// traffic is one 64 KB read per CTA per tile, half the HBM traffic.
//   M:  out = x + i t1 y              (one exchange)
//   P:  out = phi_m v (1 + i t2 K)    (H|0> is uniform: no exchange)
#pragma once
#include "lrq_sweep_wd.cuh"

namespace lrq {

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(unsigned saddr, unsigned rank) {
  unsigned d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on an mbarrier of another CTA of the cluster (release: this
// thread's earlier shared-memory writes are visible to the waiter)
__device__ __forceinline__ void mbar_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity), "r"(2000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, unsigned parity) {
  if (mbar_try_wait_cluster(b, parity)) return;
  const unsigned long long t0 = global_ns();
  while (!mbar_try_wait_cluster(b, parity))
    if (global_ns() - t0 > kMbarTrapNs) __trap();
}
__device__ __forceinline__ float4 ld_cluster_f4(unsigned cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

constexpr int kWdcBarriers = kWdTeamsMax * kWdWarps * 2;  // [team][warp][ready, done]

__host__ __device__ inline size_t wdc_smem_bytes(int n, int nst, bool usesJ) {
  return wd_smem_bytes(n, nst, usesJ) + 8 * (size_t)kWdTT + 8 * 64 + 8 * kWdcBarriers + 64;
}

template <int GK, int SK, int TEAMS>
__global__ void __launch_bounds__(TEAMS* kWdWarps * 32, 1) sweep_wdc_kernel(const __grid_constant__ SweepParams P) {
  typedef float T;
  typedef WdSweep<T, GK, SK> W;
  constexpr int kWdThreads = TEAMS * kWdWarps * 32;
  typedef typename W::U U;
  constexpr int MA = W::MA, MU = W::MU, KA = W::KA, RA = W::RA, NV = W::NV;
  constexpr bool PH = W::PH, INIT = W::INIT;
  static_assert(SK == SK_M || SK == SK_F || SK == SK_P, "cluster sweeps: P, M, F");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const unsigned smem_off = (1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u;
  unsigned char* smem = smem_raw + smem_off;

  const int n = P.n, q0 = P.q0, qU = q0 - 1;
  const int nst = P.nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned crank = cluster_rank(), prank = crank ^ 1u;
  const int cq = q0 + KA - MA;  // the cross qubit: the bit above the half tile
  const double sgn_c = crank ? -1.0 : 1.0;
  unsigned char* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nst * kWdStageBytes);
  unsigned char* sp = smem + (size_t)nst * kWdStageBytes + 128;
  double *Jm = nullptr, *Jx = nullptr;
  if (PH) {
    Jm = reinterpret_cast<double*>(sp);
    Jx = Jm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  double* thr = reinterpret_cast<double*>(sp);
  void* PRR = reinterpret_cast<void*>(thr + (kWdRAmax + 1) * kWdTT);
  double* wsc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(PRR) + 16 * 64);
  int* blk = reinterpret_cast<int*>(wsc + kWdTeamsMax * 16);
  double* Tc = reinterpret_cast<double*>(blk + 64);   // [kWdTT] thread part of h_c
  float2* GRR = reinterpret_cast<float2*>(Tc + kWdTT);  // [64] exp(2 i s_c (register part of h_c))
  uint64_t* xbar = reinterpret_cast<uint64_t*>(GRR + 64);  // [team][warp][2]
  LRQ_CHECK_SMEM(smem_raw, xbar + kWdcBarriers);
  LRQ_CHECK((gridDim.x & 1) == 0 && cq < n && (P.num_tiles & 1) == 0);
  int nb = 0;
  for (int j = 0; j < n; ++j)
    if (j >= MA && !(j >= q0 && j < q0 + KA - MA)) ++nb;

  const int bl = qU - MU;  // block unit bits below the high run
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s)
      for (int t = 0; t < TEAMS; ++t) mbar_init(&full[s * TEAMS + t], 1);
    for (int i = 0; i < kWdcBarriers; ++i) mbar_init(&xbar[i], 1);
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
    // per tile-thread constants of the phase layout (L2), as in sweep_wd_kernel,
    // plus Tc: the thread bits' part of the field on the cross qubit
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
      double ett = 0.0, tc = 0.0;
      for (int j = 0; j < 7; ++j) {
        const int gj = W::gpos(W::thr_bit(2, j), q0);
        const double sj = ((tt >> j) & 1) ? -1.0 : 1.0;
        tc += sj * Jm[cq * n + gj];
        for (int j2 = j + 1; j2 < 7; ++j2) {
          const double w = Jm[gj * n + W::gpos(W::thr_bit(2, j2), q0)];
          ett += (((tt >> j2) & 1) ? -sj : sj) * w;
        }
      }
      thr[RA * kWdTT + tt] = ett;
      Tc[tt] = tc;
    }
    for (int v = threadIdx.x; v < NV; v += kWdThreads) {
      double acc = 0.0, g = 0.0;
      for (int a = 0; a < RA; ++a) {
        const int ga = W::gpos(W::reg_bit(2, a), q0);
        const double sa = ((v >> a) & 1) ? -1.0 : 1.0;
        g += sa * Jm[cq * n + ga];
        for (int b = a + 1; b < RA; ++b) {
          const double w = Jm[ga * n + W::gpos(W::reg_bit(2, b), q0)];
          acc += (((v >> b) & 1) ? -sa : sa) * w;
        }
      }
      reinterpret_cast<float2*>(PRR)[v] = phasor32(acc);
      GRR[v] = phasor32(-2.0 * sgn_c * g);  // exp(+2 i s_c g)
    }
  }
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers are initialised before any remote arrive

  // tile of the k-th step of this CTA: pair tile ptid, half `crank` (the
  // cross qubit is the lowest tile-index bit above the block bits below q0)
  const long long nclusters = gridDim.x >> 1, cid = blockIdx.x >> 1;
  const long long pairs = P.num_tiles >> 1;
  auto tile_of = [&](long long k) -> long long {
    const long long pt = cid + k * nclusters;
    if (pt >= pairs) return -1;
    const long long lo = pt & ((1ll << bl) - 1);
    return (((pt >> bl) << 1 | (long long)crank) << bl) | lo;
  };
  auto feed = [&](int s, long long k) {
    const long long tid = tile_of(k);
    if (tid < 0) return;
    uint64_t* fb = &full[s * TEAMS + (int)(k % TEAMS)];
    if constexpr (INIT) {
      mbar_arrive(fb);
    } else {
      void* dst = stages + (size_t)s * kWdStageBytes;
      mbar_expect_tx(fb, kStageBytes);
      const int c1 = (int)((uint64_t)tid & ((1ull << bl) - 1ull)), c4 = (int)((uint64_t)tid >> bl);
      tma_load_5d(dst, &P.tmap, fb, 0, 0, c1, 0, c4);
    }
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < nst; ++s) feed(s, s);

  const int team = warp / kWdWarps, wq = warp % kWdWarps;
  const int tt2 = wq | (lane << 2);
  double* hb = wsc + team * 16;  // hb[0..KA-1] fields, hb[13] field on the cross qubit, hb[15] block energy
  U r[32];
  constexpr int RPH = INIT ? 0 : 1;
  const double2 scale = make_double2(P.scale_re, P.scale_im);
  const float t1 = (float)P.tc[0], t2 = (float)P.tc[1];
  const float2 tv1 = make_float2(-t1, t1), tv2 = make_float2(-t2, t2);
  uint64_t* xr = &xbar[(team * kWdWarps + wq) * 2 + 0];  // partner's region is ready
  uint64_t* xd = &xbar[(team * kWdWarps + wq) * 2 + 1];  // partner has read my region
  const unsigned xr_remote = mapa(smem_u32(xr), prank), xd_remote = mapa(smem_u32(xd), prank);

  long long j = 0;  // this team's tile counter (barrier parity)
  for (long long k = team;; k += TEAMS, ++j) {
    const long long tid = tile_of(k);
    if (tid < 0) break;
    const int s = (int)(k % nst);
    U* st = reinterpret_cast<U*>(stages + (size_t)s * kWdStageBytes);
    U* rg = st + wq * kWdRegion;
    const uint64_t ut = (uint64_t)tid;
    const uint64_t baseU = ((ut & ((1ull << bl) - 1ull)) << MU) | ((ut >> bl) << (qU + kUnitBits - MU));

    if constexpr (PH) {
      if (wq == 0) {
        const uint64_t base = baseU << 1;
        if (lane < KA || lane == 13) {
          const int gi = lane < KA ? W::gpos(lane, q0) : cq;
          double acc = Jx[gi];
          for (int m = 0; m < nb; ++m) acc = fma(Jm[gi * n + blk[m]], spin(base, blk[m]), acc);
          hb[lane] = acc;
        }
        double term = 0.0;
        for (int m = lane; m < nb; m += 32) {
          const int jj = blk[m];
          double fj = 0.0;
          for (int m2 = 0; m2 < nb; ++m2) fj = fma(Jm[jj * n + blk[m2]], spin(base, blk[m2]), fj);
          term += spin(base, jj) * (Jx[jj] + 0.5 * fj);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
        if (lane == 0) hb[15] = P.J.cst + term;
      }
    }

    mbar_wait(&full[s * TEAMS + team], (unsigned)((k / (nst % TEAMS == 0 ? nst : nst * TEAMS)) & 1));
    if constexpr (!INIT) {
#pragma unroll
      for (int b = 0; b < 32; ++b) r[b] = st[W::nat(wq, lane, b)];
      if (!PH && !(scale.x == 1.0 && scale.y == 0.0)) W::scale_all(r, scale);
      W::template mix<31u>(r, P.tf[0][0], P.td[0][0]);
      team_sync_n(1 + team, kWdWarps * 32);
#pragma unroll
      for (int b = 0; b < 32; ++b) rg[W::slot(lane, b)] = r[b];
      __syncwarp();
#pragma unroll
      for (int a = 0; a < 32; ++a) r[a] = rg[W::slot(a, lane)];
      W::template mix<W::L2MASK>(r, P.tf[0][1], P.td[0][1]);
      // ---- exchange with the partner CTA: my post-mix1 values into my
      // region (each lane rewrites only the slots it just read), the
      // partner's from its region
#pragma unroll
      for (int a = 0; a < 32; ++a) rg[W::slot(a, lane)] = r[a];
      // one arrive per warp: __syncwarp orders the lanes' writes before lane
      // 0's cluster-scope release
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(xr_remote);
      mbar_wait_cluster(xr, (unsigned)(j & 1));
      const unsigned pbase = mapa(smem_u32(rg), prank);
      // the partner's values in chunks of 8 units (8 DSMEM loads in flight,
      // 32 registers: the 32 own units already hold 128)
      float2 K = make_float2(1.f, 0.f);
      if constexpr (SK == SK_F) K = phasor32(-2.0 * sgn_c * (hb[13] + Tc[tt2]));
#pragma unroll
      for (int a0 = 0; a0 < 32; a0 += 8) {
        float4 y[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) y[a] = ld_cluster_f4(pbase + 16u * (unsigned)W::slot(a0 + a, lane));
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          float2 xa[2] = {make_float2(r[a0 + a].x, r[a0 + a].y), make_float2(r[a0 + a].z, r[a0 + a].w)};
          const float2 ya[2] = {make_float2(y[a].x, y[a].y), make_float2(y[a].z, y[a].w)};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 av = bf_half(xa[h], ya[h], tv1);
            if constexpr (SK == SK_M) {
              xa[h] = av;  // M: x + i t1 y
            } else {
              // F: (x + i t1 y) + i t2 K (y + i t1 x); the phase then multiplies by phi_m
              const float2 bv = bf_half(ya[h], xa[h], tv1);
              const float2 q = cmul32(cmul32(K, GRR[2 * (a0 + a) + h]), bv);
              xa[h] = bf_half(av, q, tv2);
            }
          }
          r[a0 + a] = make_float4(xa[0].x, xa[0].y, xa[1].x, xa[1].y);
        }
      }
      __syncwarp();  // every lane has its partner values (they are in use above)
      if (lane == 0) mbar_arrive_remote(xd_remote);  // the partner's region may be reused
    } else {
      team_sync_n(1 + team, kWdWarps * 32);
      // P: amplitude = phi_m v (1 + i t2 K); the (1 + i t2 K) factor first,
      // the phase (with v folded into its scale) multiplies it below
      const double Kang = -2.0 * sgn_c * (hb[13] + Tc[tt2]);
      const float2 K = phasor32(Kang);
#pragma unroll
      for (int a = 0; a < 32; ++a) {
        const float2 o0 = bf_half(make_float2(1.f, 0.f), cmul32(K, GRR[2 * a]), tv2);
        const float2 o1 = bf_half(make_float2(1.f, 0.f), cmul32(K, GRR[2 * a + 1]), tv2);
        r[a] = make_float4(o0.x, o0.y, o1.x, o1.y);
      }
    }

    if constexpr (PH) {
      double C = hb[15] + thr[RA * kWdTT + tt2];
#pragma unroll
      for (int jb = 0; jb < 7; ++jb) {
        const double h = hb[W::thr_bit(2, jb)];
        C += ((tt2 >> jb) & 1) ? -h : h;
      }
      double F[RA];
#pragma unroll
      for (int a = 0; a < RA; ++a) F[a] = hb[W::reg_bit(2, a)] + thr[a * kWdTT + tt2];
      const double2 sc = INIT ? cmul(scale, make_double2(P.init_re, P.init_im)) : scale;
      WdSweep<T, GK, SK_F>::phase(r, C, F, sc, PRR);  // multiplies (never the INIT overwrite)
      W::template mix<W::L2MASK>(r, P.tf[1][RPH], P.td[1][RPH]);
    }
    // back to L1 through the region; the partner must have read it first
    if constexpr (!INIT) mbar_wait_cluster(xd, (unsigned)(j & 1));
    __syncwarp();
#pragma unroll
    for (int a = 0; a < 32; ++a) rg[W::slot(a, lane)] = r[a];
    __syncwarp();
#pragma unroll
    for (int b = 0; b < 32; ++b) r[b] = rg[W::slot(lane, b)];
    if constexpr (PH) W::template mix<31u>(r, P.tf[1][RPH + 1], P.td[1][RPH + 1]);
    team_sync_n(1 + team, kWdWarps * 32);
#pragma unroll
    for (int b = 0; b < 32; ++b) st[W::nat(wq, lane, b)] = r[b];
    fence_proxy_async();
    team_sync_n(1 + team, kWdWarps * 32);
    if (wq == kWdWarps - 1 && lane == 0) {
      const int c1 = (int)((uint64_t)tid & ((1ull << bl) - 1ull)), c4 = (int)((uint64_t)tid >> bl);
      tma_store_5d(&P.tmap, st, 0, 0, c1, 0, c4);
      bulk_commit();
      bulk_wait_read<0>();
      feed(s, k + nst);
    }
  }
  if (lane == 0) bulk_wait<0>();
  // neither CTA leaves while the partner may still read its shared memory or
  // arrive on its barriers
  cluster_sync_all();
}

}  // namespace lrq
