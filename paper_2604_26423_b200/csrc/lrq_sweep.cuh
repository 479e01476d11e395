// The tiled sweep kernel: one HBM round trip of the state applies, to every
// 2^K-amplitude tile, a short program of
//     [init | load] [mixer beta_1 on the group's qubits] [cost phase J]
//     [mixer beta_2 on the group's qubits] [final reductions] [store]
// (DESIGN.md §3.2).  Each thread keeps 2^RB amplitudes in registers; the
// butterflies of RB qubits run in registers, and shared memory only transposes
// the tile between register layouts ("rounds").
//
// Reference operations fused here (lrqbench):
//   RZZ per edge  engine.py:147-155  -> exp(-i E_J(z)), E_J built per tile
//   RX per qubit  engine.py:137-144  -> scaled butterfly x + i t y
//   H layer       engine.py:128-134  -> init value v_n (no load at all)
//   probabilities/expected_r/cut_values_range  engine.py:94-96,214-226;
//                 problem.py:158-171 -> per-tile sum p, sum p*E_w, min E_w
#pragma once
#include "lrq_device.cuh"

namespace lrq {

constexpr int kMaxRounds = 8;

enum SweepFlags : uint32_t {
  SW_INIT = 1u,    // every amplitude starts at (init_re, init_im); no load
  SW_STORE = 2u,   // write the tile back
  SW_PHASE = 4u,   // one round applies exp(-i E_J)
  SW_REDUCE = 8u,  // one round accumulates p, p*E_W, min E_W
  SW_NOAMPS = 16u  // no state at all (exhaustive max-cut search)
};
enum RoundFlags : uint8_t { RD_PHASE = 1, RD_REDUCE = 2 };

struct Round {
  int8_t lo;       // register bits = tile bits [lo, lo+RB)
  uint8_t m1, m2;  // register bits that take a mixer-1 / mixer-2 butterfly
  uint8_t flags;   // RD_PHASE (between m1 and m2), RD_REDUCE (after m2)
};

struct MatArg {
  const double* M;    // n*n symmetric, zero diagonal, physical bit order
  const double* ext;  // n: field from bits outside this shard (global qubits)
  double cst;         // constant from bits outside this shard
};

struct SweepParams {
  void* amps;
  int n, m, q0;
  long long num_tiles;
  int nrounds;
  Round rounds[kMaxRounds];
  int store_lo;
  uint32_t flags;
  double t1, t2;
  int swap1, swap2;
  double scale_re, scale_im;
  double init_re, init_im;
  MatArg J, W;
  int min_bit;  // local bit that must be 0 for the min-E search (-1: none, -2: skip all)
  double* red_p;
  double* red_pE;
  double* red_minE;
  unsigned long long* red_arg;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// dynamic shared memory needed by sweep_kernel<T, NTB, RB>
__host__ __device__ inline size_t sweep_smem_bytes(int vbytes, int NTB, int RB, int n, uint32_t flags) {
  const int K = NTB + RB, NT = 1 << NTB, NV = 1 << RB;
  size_t b = 0;
  if (!(flags & SW_NOAMPS)) b += (size_t)vbytes << K;
  if (flags & SW_PHASE) b = align16(b + 8 * (size_t)(n * n + n));
  if (flags & SW_REDUCE) b = align16(b + 8 * (size_t)(n * n + n));
  b += 8 * (size_t)(2 * 2 * K + 4);
  b += 8 * (size_t)(2 * (RB + 1) * NT);
  b = align16(b);
  b += 16 * (size_t)NV + 8 * (size_t)NV;
  b += 8 * 4 * (size_t)(NT / 32);
  return align16(b);
}

template <typename T, int NTB, int RB>
struct Sweep {
  static constexpr int NT = 1 << NTB, K = NTB + RB, NV = 1 << RB, NW = NT / 32;
  typedef typename CxT<T>::V V;
  static constexpr int SWM = 128 / (int)sizeof(V) - 1;

  __device__ static __forceinline__ int gpos(int i, int m, int q0) { return i < m ? i : q0 + (i - m); }
  __device__ static __forceinline__ int tbit(int j, int lo) { return j < lo ? j : j + RB; }
  __device__ static __forceinline__ unsigned ebase(unsigned t, int lo) {
    return (t & ((1u << lo) - 1u)) | ((t >> lo) << (lo + RB));
  }
  __device__ static __forceinline__ unsigned swz(unsigned e) { return e ^ ((e >> RB) & SWM); }
  __device__ static __forceinline__ uint64_t gmap(unsigned e, int m, int q0) {
    return (uint64_t)(e & ((1u << m) - 1u)) | ((uint64_t)(e >> m) << q0);
  }
  __device__ static __forceinline__ bool blockbit(int j, int m, int q0, int K_) {
    return j >= m && !(j >= q0 && j < q0 + K_ - m);
  }

  // per-thread constants of layout lo for matrix M: T_a (a<RB) and E_TT
  __device__ static void thread_consts(const double* M, int n, int m, int q0, int lo, unsigned t, double* dst) {
    for (int a = 0; a < RB; ++a) {
      const int ga = gpos(lo + a, m, q0);
      double acc = 0.0;
      for (int j = 0; j < NTB; ++j) {
        const double w = M[ga * n + gpos(tbit(j, lo), m, q0)];
        acc += ((t >> j) & 1u) ? -w : w;
      }
      dst[a * NT + t] = acc;
    }
    double ett = 0.0;
    for (int j = 0; j < NTB; ++j) {
      const int gj = gpos(tbit(j, lo), m, q0);
      const double sj = ((t >> j) & 1u) ? -1.0 : 1.0;
      for (int j2 = j + 1; j2 < NTB; ++j2) {
        const double w = M[gj * n + gpos(tbit(j2, lo), m, q0)];
        ett += (((t >> j2) & 1u) ? -sj : sj) * w;
      }
    }
    dst[RB * NT + t] = ett;
  }

  // E over the register bits only, for pattern v (thread v < NV)
  __device__ static double err_entry(const double* M, int n, int m, int q0, int lo, unsigned v) {
    double acc = 0.0;
    for (int a = 0; a < RB; ++a) {
      const int ga = gpos(lo + a, m, q0);
      const double sa = ((v >> a) & 1u) ? -1.0 : 1.0;
      for (int b = a + 1; b < RB; ++b) {
        const double w = M[ga * n + gpos(lo + b, m, q0)];
        acc += (((v >> b) & 1u) ? -sa : sa) * w;
      }
    }
    return acc;
  }

  // block (tile) constants: field on each tile bit from the tile's fixed bits,
  // and the energy of the fixed bits.  Uses warps w0 (fields) and w0+1 (energy).
  __device__ static void block_consts(const double* M, const double* X, double cst, int n, int m, int q0,
                                      uint64_t base, int w0, double* hb, double* ebb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == w0) {
      if (lane < K) {
        const int gi = gpos(lane, m, q0);
        double acc = X[gi];
        for (int j = 0; j < n; ++j)
          if (blockbit(j, m, q0, K)) acc += M[gi * n + j] * spin(base, j);
        hb[lane] = acc;
      }
    } else if (warp == w0 + 1) {
      double term = 0.0;
      for (int j = lane; j < n; j += 32) {
        if (!blockbit(j, m, q0, K)) continue;
        double f = 0.0;
        for (int l = 0; l < n; ++l)
          if (blockbit(l, m, q0, K)) f += M[j * n + l] * spin(base, l);
        term += spin(base, j) * (X[j] + 0.5 * f);
      }
      for (int o = 16; o > 0; o >>= 1) term += __shfl_xor_sync(0xffffffffu, term, o);
      if (lane == 0) *ebb = cst + term;
    }
  }

  template <bool SWAP>
  __device__ static __forceinline__ void mix_impl(V (&a)[NV], unsigned mask, T t) {
    typedef typename CxT<T>::V VV;
#pragma unroll
    for (int b = 0; b < RB; ++b) {
      if (!((mask >> b) & 1u)) continue;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if ((v >> b) & 1) continue;
        const int u = v | (1 << b);
        const VV x = a[v], y = a[u];
        VV nx, ny;
        if constexpr (sizeof(T) == 4) {
          const float2 tv = make_float2(-(float)t, (float)t);
          nx = bf_half(x, y, tv);
          ny = bf_half(y, x, tv);
        } else {
          nx = bf_half(x, y, (double)t);
          ny = bf_half(y, x, (double)t);
        }
        a[v] = SWAP ? ny : nx;
        a[u] = SWAP ? nx : ny;
      }
    }
  }
  __device__ static __forceinline__ void mix(V (&a)[NV], unsigned mask, double t, int swap) {
    if (swap) mix_impl<true>(a, mask, (T)t);
    else mix_impl<false>(a, mask, (T)t);
  }
};

template <typename T, int NTB, int RB>
__global__ void __launch_bounds__(1 << NTB, 2) sweep_kernel(const SweepParams P) {
  typedef Sweep<T, NTB, RB> S;
  constexpr int NT = S::NT, K = S::K, NV = S::NV, NW = S::NW;
  typedef typename S::V V;
  extern __shared__ __align__(16) unsigned char smem[];

  const int n = P.n, m = P.m, q0 = P.q0;
  const unsigned t = threadIdx.x;
  const uint32_t flags = P.flags;
  const bool noamps = flags & SW_NOAMPS;
  const bool usesJ = flags & SW_PHASE, usesW = flags & SW_REDUCE;

  unsigned char* sp = smem;
  V* tile = reinterpret_cast<V*>(sp);
  if (!noamps) sp += sizeof(V) << K;
  double *Jm = nullptr, *Jx = nullptr, *Wm = nullptr, *Wx = nullptr;
  if (usesJ) {
    Jm = reinterpret_cast<double*>(sp);
    Jx = Jm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  if (usesW) {
    Wm = reinterpret_cast<double*>(sp);
    Wx = Wm + n * n;
    sp = smem + align16((size_t)(sp - smem) + 8 * (size_t)(n * n + n));
  }
  double* hB = reinterpret_cast<double*>(sp);  // [parity][mat][K]
  double* EBB = hB + 2 * 2 * K;                // [parity][mat]
  double* thr = EBB + 4;                       // [mat][(RB+1)][NT]
  sp = smem + align16((size_t)(reinterpret_cast<unsigned char*>(thr + 2 * (RB + 1) * NT) - smem));
  double2* PRR = reinterpret_cast<double2*>(sp);
  double* ERR = reinterpret_cast<double*>(PRR + NV);
  double* rs = ERR + NV;  // [NW][4]

  for (int i = t; i < n * n; i += NT) {
    if (usesJ) Jm[i] = P.J.M[i];
    if (usesW) Wm[i] = P.W.M[i];
  }
  for (int i = t; i < n; i += NT) {
    if (usesJ) Jx[i] = P.J.ext[i];
    if (usesW) Wx[i] = P.W.ext[i];
  }
  int lo_phase = -1, lo_red = -1;
  for (int r = 0; r < P.nrounds; ++r) {
    if (P.rounds[r].flags & RD_PHASE) lo_phase = P.rounds[r].lo;
    if (P.rounds[r].flags & RD_REDUCE) lo_red = P.rounds[r].lo;
  }
  __syncthreads();
  if (usesJ) {
    S::thread_consts(Jm, n, m, q0, lo_phase, t, thr);
    if (t < NV) PRR[t] = expmi(S::err_entry(Jm, n, m, q0, lo_phase, t));
  }
  if (usesW) {
    S::thread_consts(Wm, n, m, q0, lo_red, t, thr + (RB + 1) * NT);
    if (t < NV) ERR[t] = S::err_entry(Wm, n, m, q0, lo_red, t);
  }

  const double2 scale = make_double2(P.scale_re, P.scale_im);
  const bool unit_scale = (P.scale_re == 1.0 && P.scale_im == 0.0);
  V* amps = reinterpret_cast<V*>(P.amps);
  const int bl = q0 - m;  // block bits below the high target run

  int par = 0;
  for (long long tid = blockIdx.x; tid < P.num_tiles; tid += gridDim.x, par ^= 1) {
    const uint64_t ut = (uint64_t)tid;
    const uint64_t base = ((ut & ((1ull << bl) - 1ull)) << m) | ((ut >> bl) << (q0 + K - m));
    double* hbJ = hB + (par * 2 + 0) * K;
    double* hbW = hB + (par * 2 + 1) * K;
    if (usesJ) S::block_consts(Jm, Jx, P.J.cst, n, m, q0, base, 0, hbJ, &EBB[par * 2 + 0]);
    if (usesW) S::block_consts(Wm, Wx, P.W.cst, n, m, q0, base, 2, hbW, &EBB[par * 2 + 1]);
    __syncthreads();

    V a[NV];
    int cur = P.rounds[0].lo;
    bool dirty = false;
    if (!noamps) {
      if (flags & SW_INIT) {
        V iv;
        iv.x = (T)P.init_re;
        iv.y = (T)P.init_im;
#pragma unroll
        for (int v = 0; v < NV; ++v) a[v] = iv;
      } else {
        const unsigned eb = S::ebase(t, cur);
        const uint64_t z0 = base + S::gmap(eb, m, q0);
        const int sh = cur >= m ? cur - m + q0 : cur;
#pragma unroll
        for (int v = 0; v < NV; ++v) a[v] = ld_amp(amps + z0 + ((uint64_t)v << sh));
      }
      if (!usesJ && !unit_scale) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (P.scale_im == 0.0) {
            a[v].x *= (T)P.scale_re;
            a[v].y *= (T)P.scale_re;
          } else {
            a[v] = cmul_amp(a[v], scale);
          }
        }
      }
    }

    for (int r = 0; r < P.nrounds; ++r) {
      const Round R = P.rounds[r];
      if (!noamps && R.lo != cur) {
        if (dirty) __syncthreads();
        const unsigned eo = S::ebase(t, cur);
#pragma unroll
        for (int v = 0; v < NV; ++v) tile[S::swz(eo + ((unsigned)v << cur))] = a[v];
        __syncthreads();
        const unsigned en = S::ebase(t, R.lo);
#pragma unroll
        for (int v = 0; v < NV; ++v) a[v] = tile[S::swz(en + ((unsigned)v << R.lo))];
        dirty = true;
        cur = R.lo;
      }
      if (R.m1) S::mix(a, R.m1, P.t1, P.swap1);
      if (R.flags & RD_PHASE) {
        const double* th = thr;
        double f[RB];
        double ang = EBB[par * 2 + 0] + th[RB * NT + t];
#pragma unroll
        for (int j = 0; j < NTB; ++j) {
          const double h = hbJ[S::tbit(j, cur)];
          ang += ((t >> j) & 1u) ? -h : h;
        }
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          f[b] = hbJ[cur + b] + th[b * NT + t];
          ang += f[b];
        }
        double2 d[RB];
#pragma unroll
        for (int b = 0; b < RB; ++b) d[b] = expmi(-2.0 * f[b]);  // exp(+2i f_b)
        double2 phi = cmul(scale, expmi(ang));
        a[0] = cmul_amp(a[0], cmul(phi, PRR[0]));
#pragma unroll
        for (int k = 1; k < NV; ++k) {
          const int b = (__ffs(k) - 1);
          const int v = k ^ (k >> 1);
          phi = ((v >> b) & 1) ? cmul(phi, d[b]) : cmul_conj(phi, d[b]);
          a[v] = cmul_amp(a[v], cmul(phi, PRR[v]));
        }
      }
      if (R.m2) S::mix(a, R.m2, P.t2, P.swap2);
      if (R.flags & RD_REDUCE) {
        const double* th = thr + (RB + 1) * NT;
        double f[RB];
        double e = EBB[par * 2 + 1] + th[RB * NT + t];
        bool thread_ok = true;
#pragma unroll
        for (int j = 0; j < NTB; ++j) {
          const int i = S::tbit(j, cur);
          const double h = hbW[i];
          const bool bit = (t >> j) & 1u;
          e += bit ? -h : h;
          if (bit && S::gpos(i, m, q0) == P.min_bit) thread_ok = false;
        }
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          f[b] = hbW[cur + b] + th[b * NT + t];
          e += f[b];
        }
        unsigned vmask = 0;  // register bit that must be 0 for the min search
#pragma unroll
        for (int b = 0; b < RB; ++b)
          if (S::gpos(cur + b, m, q0) == P.min_bit) vmask = 1u << b;
        if (P.min_bit == -2 || (P.min_bit >= 0 && ((base >> P.min_bit) & 1ull))) thread_ok = false;

        double sp_ = 0.0, spe = 0.0, mine = __longlong_as_double(0x7ff0000000000000ll);
        int bestv = NV;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
          const int v = k ^ (k >> 1);
          if (k) {
            const int b = (__ffs(k) - 1);
            e += ((v >> b) & 1) ? -2.0 * f[b] : 2.0 * f[b];
          }
          const double ev = e + ERR[v];
          if (!noamps) {
            const double pv = prob(a[v]);
            sp_ += pv;
            spe = fma(pv, ev, spe);
          }
          if (thread_ok && !(v & vmask) && (ev < mine || (ev == mine && v < bestv))) {
            mine = ev;
            bestv = v;
          }
        }
        const int sh = cur >= m ? cur - m + q0 : cur;
        unsigned long long zbest = ~0ull;
        if (bestv < NV) zbest = base + S::gmap(S::ebase(t, cur), m, q0) + ((uint64_t)bestv << sh);
        // deterministic warp tree, then fixed-order combine of the warps
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sp_ += __shfl_xor_sync(0xffffffffu, sp_, o);
          spe += __shfl_xor_sync(0xffffffffu, spe, o);
          const double om = __shfl_xor_sync(0xffffffffu, mine, o);
          const unsigned long long oz = __shfl_xor_sync(0xffffffffu, zbest, o);
          if (om < mine || (om == mine && oz < zbest)) {
            mine = om;
            zbest = oz;
          }
        }
        const int warp = t >> 5;
        if ((t & 31) == 0) {
          rs[warp * 4 + 0] = sp_;
          rs[warp * 4 + 1] = spe;
          rs[warp * 4 + 2] = mine;
          rs[warp * 4 + 3] = __longlong_as_double((long long)zbest);
        }
        __syncthreads();
        if (t == 0) {
          double s0 = 0.0, s1 = 0.0, mn = rs[2];
          unsigned long long zb = (unsigned long long)__double_as_longlong(rs[3]);
          for (int w = 0; w < NW; ++w) {
            s0 += rs[w * 4 + 0];
            s1 += rs[w * 4 + 1];
            const double om = rs[w * 4 + 2];
            const unsigned long long oz = (unsigned long long)__double_as_longlong(rs[w * 4 + 3]);
            if (om < mn || (om == mn && oz < zb)) {
              mn = om;
              zb = oz;
            }
          }
          P.red_p[tid] = s0;
          P.red_pE[tid] = s1;
          P.red_minE[tid] = mn;
          P.red_arg[tid] = zb;
        }
      }
    }

    if (!noamps && (flags & SW_STORE)) {
      if (P.store_lo != cur) {
        if (dirty) __syncthreads();
        const unsigned eo = S::ebase(t, cur);
#pragma unroll
        for (int v = 0; v < NV; ++v) tile[S::swz(eo + ((unsigned)v << cur))] = a[v];
        __syncthreads();
        cur = P.store_lo;
        const unsigned en = S::ebase(t, cur);
#pragma unroll
        for (int v = 0; v < NV; ++v) a[v] = tile[S::swz(en + ((unsigned)v << cur))];
      }
      const unsigned eb = S::ebase(t, cur);
      const uint64_t z0 = base + S::gmap(eb, m, q0);
      const int sh = cur >= m ? cur - m + q0 : cur;
#pragma unroll
      for (int v = 0; v < NV; ++v) st_amp(amps + z0 + ((uint64_t)v << sh), a[v]);
    }
  }
}

}  // namespace lrq
