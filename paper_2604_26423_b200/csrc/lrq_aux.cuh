// Auxiliary kernels: whole-state path for tiny n, deterministic finalisation
// of the per-tile reductions (+ CDF block prefix), the two-level inverse-CDF
// sampler, and the bit-exact sequential cut diagonal.
#pragma once
#include "lrq_device.cuh"

namespace lrq {

// ---------------------------------------------------------------------------
// n < K: the whole circuit in one CTA, state in shared memory.
// Same operations as the sweep path (phase exp(-i E_J), RX butterflies),
// written plainly: tiny n is a correctness path, not a performance one.
struct SmallParams {
  void* amps;
  int n, p;
  const double* J;    // p * n * n
  const double* mix;  // p * 2: (cos h, -sin h) of RX(theta), h = theta / 2
  const double* W;    // n * n cost matrix (may be null: no reduction)
  const double* F;    // p * n single-Z fields (may be null)
  const double* Fc;   // p constant phases (with F)
  // batched noisy trajectories (lrq_noisy_batch): block b runs trajectory b
  // with its own J (b * strideJ), per-qubit mixer signs msign[b*p*n + k*n + q]
  // (sin h -> -sin h where negative; null: all +), and writes the trajectory's
  // probabilities, index-permuted by its Pauli X mask, to probs[b * 2^n + ...]
  const signed char* msign;
  long long strideJ;
  const unsigned* xmask;
  double* probs;
  double init_re, init_im;
  int load;  // start from the stored state instead of the init value
  int min_bit;
  double* red_p;
  double* red_pE;
  double* red_minE;
  unsigned long long* red_arg;
  double* red_maxE;              // may be null
  int search;                    // unused here: the whole-state path always searches (tiny n)
  unsigned long long* hist;      // global energy histogram (may be null), see SweepParams
  int hist_bins;
  double hist_lo, hist_scale;
};

template <typename T>
__global__ void __launch_bounds__(256) small_kernel(const SmallParams P) {
  typedef typename CxT<T>::V V;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = P.n, N = 1 << n;
  V* s = reinterpret_cast<V*>(smem);
  double* red = reinterpret_cast<double*>(s + N);  // 8 warps * 5
  LRQ_CHECK_SMEM(smem, red + 5 * (blockDim.x >> 5));
  const int t = threadIdx.x;
  const int b = blockIdx.x;  // trajectory (batch); 0 for a single state
  const V* g0 = reinterpret_cast<const V*>(P.amps);
  for (int z = t; z < N; z += blockDim.x) {
    if (P.load) {
      s[z] = g0[z];
    } else {
      s[z].x = (T)P.init_re;
      s[z].y = (T)P.init_im;
    }
  }
  __syncthreads();
  const signed char* msign = P.msign ? P.msign + (size_t)b * P.p * n : nullptr;
  for (int k = 0; k < P.p; ++k) {
    const double* J = P.J + (size_t)b * P.strideJ + (size_t)k * n * n;
    for (int z = t; z < N; z += blockDim.x) {
      double e = 0.0;
      for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) e += J[i * n + j] * spin(z, i) * spin(z, j);
      if (P.F) {
        for (int i = 0; i < n; ++i) e += P.F[(size_t)k * n + i] * spin(z, i);
        e += P.Fc[k];
      }
      s[z] = cmul_amp(s[z], expmi(e));
    }
    __syncthreads();
    const T c = (T)P.mix[2 * k], sn0 = (T)P.mix[2 * k + 1];
    for (int q = 0; q < n; ++q) {
      const T sn = (msign && msign[k * n + q] < 0) ? -sn0 : sn0;
      for (int pi = t; pi < N / 2; pi += blockDim.x) {
        const int lo = ((pi >> q) << (q + 1)) | (pi & ((1 << q) - 1));
        const int hi = lo | (1 << q);
        const V x = s[lo], y = s[hi];
        V nx, ny;  // c x + i sn y
        nx.x = c * x.x - sn * y.y;
        nx.y = c * x.y + sn * y.x;
        ny.x = c * y.x - sn * x.y;
        ny.y = c * y.y + sn * x.x;
        s[lo] = nx;
        s[hi] = ny;
      }
      __syncthreads();
    }
  }
  if (P.probs) {
    const unsigned m = P.xmask ? P.xmask[b] : 0u;
    double* out = P.probs + (size_t)b * N;
    for (int z = t; z < N; z += blockDim.x) out[z ^ m] = prob(s[z]);
    return;
  }
  V* g = reinterpret_cast<V*>(P.amps);
  for (int z = t; z < N; z += blockDim.x) g[z] = s[z];
  if (P.W == nullptr) return;
  double sp = 0.0, spe = 0.0, mine = __longlong_as_double(0x7ff0000000000000ll);
  double maxe = -mine;
  unsigned long long zb = ~0ull;
  for (int z = t; z < N; z += blockDim.x) {
    double e = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) e += P.W[i * n + j] * spin(z, i) * spin(z, j);
    const double pv = prob(s[z]);
    sp += pv;
    spe = fma(pv, e, spe);
    maxe = fmax(maxe, e);
    if (P.hist) hist_add(P.hist, P.hist_bins, P.hist_lo, P.hist_scale, e, pv);
    const bool ok = P.min_bit == -1 || (P.min_bit >= 0 && !((z >> P.min_bit) & 1));
    if (ok && (e < mine || (e == mine && (unsigned long long)z < zb))) {
      mine = e;
      zb = z;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    sp += __shfl_xor_sync(0xffffffffu, sp, o);
    spe += __shfl_xor_sync(0xffffffffu, spe, o);
    const double om = __shfl_xor_sync(0xffffffffu, mine, o);
    const unsigned long long oz = __shfl_xor_sync(0xffffffffu, zb, o);
    if (om < mine || (om == mine && oz < zb)) {
      mine = om;
      zb = oz;
    }
    maxe = fmax(maxe, __shfl_xor_sync(0xffffffffu, maxe, o));
  }
  if ((t & 31) == 0) {
    red[(t >> 5) * 5 + 0] = sp;
    red[(t >> 5) * 5 + 1] = spe;
    red[(t >> 5) * 5 + 2] = mine;
    red[(t >> 5) * 5 + 3] = __longlong_as_double((long long)zb);
    red[(t >> 5) * 5 + 4] = maxe;
  }
  __syncthreads();
  if (t == 0) {
    double s0 = 0.0, s1 = 0.0, mn = red[2], mx = red[4];
    unsigned long long b = (unsigned long long)__double_as_longlong(red[3]);
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      s0 += red[w * 5];
      s1 += red[w * 5 + 1];
      const double om = red[w * 5 + 2];
      const unsigned long long oz = (unsigned long long)__double_as_longlong(red[w * 5 + 3]);
      if (om < mn || (om == mn && oz < b)) {
        mn = om;
        b = oz;
      }
      mx = fmax(mx, red[w * 5 + 4]);
    }
    P.red_p[0] = s0;
    P.red_pE[0] = s1;
    P.red_minE[0] = mn;
    P.red_arg[0] = b;
    if (P.red_maxE) P.red_maxE[0] = mx;
  }
}

// ---------------------------------------------------------------------------
// Deterministic combine of the per-tile partials + exclusive CDF prefix over
// tiles.  One CTA; each thread owns a contiguous run of tiles; fixed order.
// out[0] = sum p, out[1] = sum p*E_w, out[2] = min E_w, out[3] = argmin (bits)
__global__ void __launch_bounds__(1024) finalize_kernel(long long T, const double* __restrict__ rp,
                                                         const double* __restrict__ rpe,
                                                         const double* __restrict__ rmin,
                                                         const unsigned long long* __restrict__ rarg,
                                                         const double* __restrict__ rmax,
                                                         double* __restrict__ prefix, double* __restrict__ out) {
  __shared__ double s_p[1024], s_pe[1024], s_min[1024], s_max[1024];
  __shared__ unsigned long long s_arg[1024];
  const int t = threadIdx.x, NTH = blockDim.x;
  const long long per = (T + NTH - 1) / NTH;
  const long long lo = min(T, per * t), hi = min(T, lo + per);
  double a = 0.0, b = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  unsigned long long z = ~0ull;
  for (long long i = lo; i < hi; ++i) {
    a += rp[i];
    b += rpe[i];
    const double m = rmin[i];
    if (m < mn || (m == mn && rarg[i] < z)) {
      mn = m;
      z = rarg[i];
    }
    mx = fmax(mx, rmax[i]);
  }
  s_p[t] = a;
  s_pe[t] = b;
  s_min[t] = mn;
  s_arg[t] = z;
  s_max[t] = mx;
  __syncthreads();
  if (t == 0) {
    double acc = 0.0, accb = 0.0, m = s_min[0], M = s_max[0];
    unsigned long long zz = s_arg[0];
    for (int i = 0; i < NTH; ++i) {
      const double x = s_p[i];
      s_p[i] = acc;  // exclusive offset of thread i
      acc += x;
      accb += s_pe[i];
      if (s_min[i] < m || (s_min[i] == m && s_arg[i] < zz)) {
        m = s_min[i];
        zz = s_arg[i];
      }
      M = fmax(M, s_max[i]);
    }
    out[0] = acc;
    out[1] = accb;
    out[2] = m;
    out[3] = __longlong_as_double((long long)zz);
    out[4] = M;
    prefix[T] = acc;
  }
  __syncthreads();
  double run = s_p[t];
  for (long long i = lo; i < hi; ++i) {
    prefix[i] = run;
    run += rp[i];
  }
}

// Multi-CTA form of finalize_kernel for large tile counts (fixed order, so
// still deterministic): pass 1 reduces block b's contiguous tile range and
// writes the block-relative exclusive prefix; pass 2 combines the block
// totals in order (out[], block offsets, prefix[T]); pass 3 adds the offsets.
constexpr int kFinBlocks = 512;
__global__ void __launch_bounds__(256) finalize_blocks(long long T, long long per_block, const double* __restrict__ rp,
                                                       const double* __restrict__ rpe,
                                                       const double* __restrict__ rmin,
                                                       const unsigned long long* __restrict__ rarg,
                                                       const double* __restrict__ rmax,
                                                       double* __restrict__ prefix, double* __restrict__ bs) {
  __shared__ double s_p[256], s_pe[256], s_min[256], s_max[256];
  __shared__ unsigned long long s_arg[256];
  const int b = blockIdx.x, t = threadIdx.x;
  const long long lo = min(T, (long long)b * per_block), hi = min(T, lo + per_block);
  const long long per_t = (hi - lo + 255) / 256;
  const long long tlo = min(hi, lo + per_t * t), thi = min(hi, tlo + per_t);
  double a = 0.0, c = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  unsigned long long z = ~0ull;
  for (long long i = tlo; i < thi; ++i) {
    a += rp[i];
    c += rpe[i];
    if (rmin[i] < mn || (rmin[i] == mn && rarg[i] < z)) {
      mn = rmin[i];
      z = rarg[i];
    }
    mx = fmax(mx, rmax[i]);
  }
  s_p[t] = a;
  s_pe[t] = c;
  s_min[t] = mn;
  s_arg[t] = z;
  s_max[t] = mx;
  __syncthreads();
  if (t == 0) {
    double acc = 0.0, accb = 0.0, m = s_min[0], M = s_max[0];
    unsigned long long zz = s_arg[0];
    for (int i = 0; i < 256; ++i) {
      const double x = s_p[i];
      s_p[i] = acc;
      acc += x;
      accb += s_pe[i];
      if (s_min[i] < m || (s_min[i] == m && s_arg[i] < zz)) {
        m = s_min[i];
        zz = s_arg[i];
      }
      M = fmax(M, s_max[i]);
    }
    bs[b] = acc;
    bs[kFinBlocks + b] = accb;
    bs[2 * kFinBlocks + b] = m;
    bs[3 * kFinBlocks + b] = __longlong_as_double((long long)zz);
    bs[5 * kFinBlocks + b] = M;
  }
  __syncthreads();
  double run = s_p[t];
  for (long long i = tlo; i < thi; ++i) {
    prefix[i] = run;
    run += rp[i];
  }
}

__global__ void finalize_combine(int nb, long long T, double* __restrict__ bs, double* __restrict__ prefix,
                                 double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double acc = 0.0, accb = 0.0, m = bs[2 * kFinBlocks], M = bs[5 * kFinBlocks];
  unsigned long long zz = (unsigned long long)__double_as_longlong(bs[3 * kFinBlocks]);
  for (int i = 0; i < nb; ++i) {
    const double x = bs[i];
    bs[4 * kFinBlocks + i] = acc;  // exclusive block offset
    acc += x;
    accb += bs[kFinBlocks + i];
    const double mi = bs[2 * kFinBlocks + i];
    const unsigned long long zi = (unsigned long long)__double_as_longlong(bs[3 * kFinBlocks + i]);
    if (mi < m || (mi == m && zi < zz)) {
      m = mi;
      zz = zi;
    }
    M = fmax(M, bs[5 * kFinBlocks + i]);
  }
  out[0] = acc;
  out[1] = accb;
  out[2] = m;
  out[3] = __longlong_as_double((long long)zz);
  out[4] = M;
  prefix[T] = acc;
}

__global__ void __launch_bounds__(256) finalize_offsets(long long T, long long per_block, const double* __restrict__ bs,
                                                        double* __restrict__ prefix) {
  const int b = blockIdx.x;
  const long long lo = min(T, (long long)b * per_block), hi = min(T, lo + per_block);
  const double off = bs[4 * kFinBlocks + b];
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) prefix[i] += off;
}

// Gate-by-gate kernels (reference engine.py:128-166, for circuits that are
// not H + p x (RZZ, RX^n)): one pass over the state per gate, with the
// reference's complex arithmetic (products and sums rounded one by one, no
// FMA contraction).  kind 0: H, 1: RX(theta).
template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void gate1q_kernel(void* amps_, int n, int q, int kind, T c, T s) {
  typedef typename CxT<T>::V V;
  V* a = reinterpret_cast<V*>(amps_);
  const long long half = 1ll << (n - 1);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < half;
       i += (long long)gridDim.x * blockDim.x) {
    const long long lo = ((i >> q) << (q + 1)) | (i & ((1ll << q) - 1));
    const long long hi = lo | (1ll << q);
    const V x = a[lo], y = a[hi];
    V u, w;
    if (kind == 0) {  // (x + y) * inv, (x - y) * inv
      u.x = mul_rn(add_rn(x.x, y.x), c);
      u.y = mul_rn(add_rn(x.y, y.y), c);
      w.x = mul_rn(add_rn(x.x, -y.x), c);
      w.y = mul_rn(add_rn(x.y, -y.y), c);
    } else if (kind == 3) {  // X: swap
      u = y;
      w = x;
    } else if (kind == 4) {  // Y: (-i y, i x)
      u.x = y.y;
      u.y = -y.x;
      w.x = -x.y;
      w.y = x.x;
    } else if (kind == 5) {  // Z: (x, -y)
      u = x;
      w.x = -y.x;
      w.y = -y.y;
    } else {  // c x + (-i s) y, (-i s) x + c y with s = sin(theta / 2)
      u.x = add_rn(mul_rn(c, x.x), mul_rn(s, y.y));
      u.y = add_rn(mul_rn(c, x.y), -mul_rn(s, y.x));
      w.x = add_rn(mul_rn(s, x.y), mul_rn(c, y.x));
      w.y = add_rn(-mul_rn(s, x.x), mul_rn(c, y.y));
    }
    a[lo] = u;
    a[hi] = w;
  }
}

// RZZ: equal bits i, j -> * e, differing -> * d (complex scalars)
template <typename T>
__global__ void rzz_kernel(void* amps_, int n, int i, int j, T er, T ei, T dr, T di) {
  typedef typename CxT<T>::V V;
  V* a = reinterpret_cast<V*>(amps_);
  const long long N = 1ll << n;
  for (long long z = blockIdx.x * (long long)blockDim.x + threadIdx.x; z < N; z += (long long)gridDim.x * blockDim.x) {
    const bool differ = ((z >> i) ^ (z >> j)) & 1;
    const T fr = differ ? dr : er, fi = differ ? di : ei;
    const V x = a[z];
    V y;
    y.x = add_rn(mul_rn(x.x, fr), -mul_rn(x.y, fi));
    y.y = add_rn(mul_rn(x.x, fi), mul_rn(x.y, fr));
    a[z] = y;
  }
}

// a[z] <-> a[z ^ mask] (each pair swapped once, by the lower index)
template <typename E>
__global__ void xor_permute_kernel(void* data, int n, unsigned long long mask) {
  E* a = reinterpret_cast<E*>(data);
  const long long N = 1ll << n;
  for (long long z = blockIdx.x * (long long)blockDim.x + threadIdx.x; z < N; z += (long long)gridDim.x * blockDim.x) {
    const long long y = z ^ (long long)mask;
    if (z < y) {
      const E t = a[z];
      a[z] = a[y];
      a[y] = t;
    }
  }
}

// |0...0> (which = 0) or the uniform value v (which = 1)
template <typename T>
__global__ void reset_kernel(void* amps_, int n, int which, T v) {
  typedef typename CxT<T>::V V;
  V* a = reinterpret_cast<V*>(amps_);
  const long long N = 1ll << n;
  for (long long z = blockIdx.x * (long long)blockDim.x + threadIdx.x; z < N; z += (long long)gridDim.x * blockDim.x) {
    V y;
    y.x = which ? v : (z == 0 ? (T)1 : (T)0);
    y.y = (T)0;
    a[z] = y;
  }
}

// Inverse-CDF draws for a batch of small distributions (noisy trajectories):
// block b owns probs[b * N ...]; cdf = sequential cumsum, normalised by its
// last element, first index with cdf > u (reference engine.py:254-263).
__global__ void __launch_bounds__(256) batch_sample_kernel(const double* __restrict__ probs, int N,
                                                           const double* __restrict__ u, long long S,
                                                           unsigned long long* __restrict__ out) {
  extern __shared__ double cdf[];
  const int b = blockIdx.x;
  const double* pr = probs + (size_t)b * N;
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int i = 0; i < N; ++i) {
      acc += pr[i];
      cdf[i] = acc;
    }
  }
  __syncthreads();
  const double total = cdf[N - 1];
  for (long long k = threadIdx.x; k < S; k += blockDim.x) {
    const double x = u[(size_t)b * S + k];
    int lo = 0, hi = N;  // first i in [0, N) with cdf[i] / total > x (N if none)
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cdf[mid] / total > x) hi = mid;
      else lo = mid + 1;
    }
    out[(size_t)b * S + k] = (unsigned long long)(lo < N ? lo : N - 1);
  }
}

// ---------------------------------------------------------------------------
// Two-level inverse-CDF sampler (reference engine.py:254-263: first index
// whose normalised cumulative probability exceeds u).  One warp per shot:
// binary search over tile prefixes, then an in-tile scan in index order.
// Src gives the probability of element e (|a_e|^2 of a state, or an explicit
// float64 distribution for draw_indices); `count` bounds a short last tile.
// Multi-GPU: this shard's CDF starts at goff of a global mass gtotal; it owns
// the uniforms in [goff, goff + its mass) / gtotal and writes 0 for the rest
// (the ranks' outputs are then summed); indices get the rank bits base_index.
template <typename T>
struct AmpProb {
  const typename CxT<T>::V* a;
  __device__ __forceinline__ double operator()(long long e) const { return prob(a[e]); }
};
struct RawProb {
  const double* p;
  __device__ __forceinline__ double operator()(long long e) const { return p[e]; }
};

template <typename Src>
__device__ __forceinline__ void sample_one(const Src& src, int tile_bits, long long T_tiles, long long count,
                                           const double* __restrict__ prefix, double x, double goff, double gtotal,
                                           unsigned long long base_index, unsigned long long* out,
                                           int write_unowned = 1) {
  const int lane = threadIdx.x & 31;
  const double total = gtotal;
  // this segment covers the cumulative mass [goff + prefix[0], goff + prefix[T_tiles])
  if (!((goff + prefix[0]) / total <= x && (goff + prefix[T_tiles]) / total > x)) {
    if (lane == 0 && write_unowned) *out = 0ull;  // one of several segments: leave the others' results
    return;
  }
  // first tile b with (goff + prefix[b+1]) / total > x
  long long lo = 0, hi = T_tiles - 1;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((goff + prefix[mid + 1]) / total > x) hi = mid;
    else lo = mid + 1;
  }
  const long long b = lo;
  LRQ_CHECK(b >= 0 && b < T_tiles);
  const long long t0 = b << tile_bits;
  const long long L = (count - t0) < (1ll << tile_bits) ? (count - t0) : (1ll << tile_bits);
  const long long chunk = (L + 31) / 32;
  const long long e0 = lane * chunk;
  const long long e1 = e0 + chunk < L ? e0 + chunk : L;
  double mine = 0.0;
  for (long long e = e0; e < e1; ++e) mine += src(t0 + e);
  // inclusive scan over lanes
  double inc = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  const double off = goff + prefix[b];
  const bool hit = e0 < L && (off + inc) / total > x;
  const unsigned ballot = __ballot_sync(0xffffffffu, hit);
  if (ballot == 0) {
    if (lane == 0) *out = base_index + (unsigned long long)(t0 + L - 1);
    return;
  }
  const int L0 = __ffs(ballot) - 1;
  if (lane == L0) {
    double c = off + inc - mine;
    long long idx = e1 - 1;
    for (long long e = e0; e < e1; ++e) {
      c += src(t0 + e);
      if (c / total > x) {
        idx = e;
        break;
      }
    }
    LRQ_CHECK(t0 + idx < count);
    *out = base_index + (unsigned long long)(t0 + idx);
  }
}

template <typename T>
__global__ void sample_kernel(const void* amps_, int tile_bits, long long T_tiles, const double* __restrict__ prefix,
                              const double* __restrict__ u, long long shots, double goff, double gtotal,
                              unsigned long long base_index, int write_unowned, unsigned long long* __restrict__ out) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (warp >= shots) return;
  AmpProb<T> src{reinterpret_cast<const typename CxT<T>::V*>(amps_)};
  sample_one(src, tile_bits, T_tiles, T_tiles << tile_bits, prefix, u[warp], goff, gtotal, base_index, out + warp,
             write_unowned);
}

// draw_indices over an explicit distribution (engine.py:254-263)
__global__ void sample_probs_kernel(const double* __restrict__ p, long long count, int tile_bits, long long T_tiles,
                                    const double* __restrict__ prefix, const double* __restrict__ u, long long shots,
                                    unsigned long long* __restrict__ out) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (warp >= shots) return;
  RawProb src{p};
  sample_one(src, tile_bits, T_tiles, count, prefix, u[warp], 0.0, prefix[T_tiles], 0ull, out + warp);
}

// per-tile sums of an explicit distribution (one warp per tile, lane chunks
// in index order, then the lane partials in lane order: deterministic)
__global__ void prob_tile_sums_kernel(const double* __restrict__ p, long long count, int tile_bits, long long T_tiles,
                                      double* __restrict__ tsum) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (warp >= T_tiles) return;
  const long long t0 = warp << tile_bits;
  const long long L = (count - t0) < (1ll << tile_bits) ? (count - t0) : (1ll << tile_bits);
  const long long chunk = (L + 31) / 32;
  const long long e0 = lane * chunk, e1 = e0 + chunk < L ? e0 + chunk : L;
  double s = 0.0;
  for (long long e = e0; e < e1; ++e) s += p[t0 + e];
  double tot = 0.0;
  for (int l = 0; l < 32; ++l) tot += __shfl_sync(0xffffffffu, s, l);
  if (lane == 0) tsum[warp] = tot;
}

// ---------------------------------------------------------------------------
// Bit-exact cut values (reference problem.py:139-149): sequential float64
// accumulation over edges in lexicographic order; w*bit is exact, and the
// adds are forced to round-to-nearest one by one (no reassociation).
__global__ void cut_values_kernel(int n, const double* __restrict__ w, const unsigned long long* __restrict__ z,
                                  long long count, unsigned long long start, double* __restrict__ out) {
  extern __shared__ double ws[];
  const int E = n * (n - 1) / 2;
  for (int i = threadIdx.x; i < E; i += blockDim.x) ws[i] = w[i];
  __syncthreads();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
       k += (long long)gridDim.x * blockDim.x) {
    const unsigned long long x = z ? z[k] : start + (unsigned long long)k;
    double acc = 0.0;
    int e = 0;
    for (int i = 0; i < n; ++i) {
      const unsigned long long xi = x >> i;
      for (int j = i + 1; j < n; ++j, ++e) {
        const unsigned long long bit = (xi ^ (x >> j)) & 1ull;
        acc = __dadd_rn(acc, bit ? ws[e] : 0.0);
      }
    }
    out[k] = acc;
  }
}


// Spin-form cut values (reference cut_values_range, problem.py:158-171):
// C(z) = W/2 - (1/4) s^T A s with s_k = 1 - 2 bit_k(z), A the symmetric weight
// matrix.  t_i = sum_j s_j A_ji (j ascending), quad = sum_i t_i s_i (i
// ascending), each add rounded in order.  The reference's own order is the
// BLAS product's, so the two agree to ~1e-15 relative, not bitwise (the
// bit-exact values are cut_values_kernel's).
__device__ __forceinline__ double cut_spin(int n, const double* __restrict__ A, double half_total,
                                           unsigned long long z) {
  double quad = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* Ai = A + i * n;
    double t = 0.0;
    for (int j = 0; j < n; ++j) t = __dadd_rn(t, ((z >> j) & 1ull) ? -Ai[j] : Ai[j]);
    quad = __dadd_rn(quad, ((z >> i) & 1ull) ? -t : t);
  }
  return __dadd_rn(half_total, -0.25 * quad);
}

__global__ void cut_values_spin_kernel(int n, const double* __restrict__ A, double half_total,
                                       unsigned long long start, long long count, double* __restrict__ out) {
  extern __shared__ double As[];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) As[i] = A[i];
  __syncthreads();
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < count;
       k += (long long)gridDim.x * blockDim.x)
    out[k] = cut_spin(n, As, half_total, start + (unsigned long long)k);
}

// expected_r_from_probs numerator (engine.py:214-226): for each 2^16 chunk c,
// sums[c] = sum_{z in chunk} p_z C_spin(z), combined in a fixed tree order
// (one CTA per chunk); the host adds the chunk sums in chunk order.
__global__ void __launch_bounds__(256) expected_cut_kernel(int n, const double* __restrict__ A, double half_total,
                                                           const double* __restrict__ p, long long count,
                                                           int chunk_bits, double* __restrict__ sums) {
  extern __shared__ double As[];
  __shared__ double part[256];
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) As[i] = A[i];
  __syncthreads();
  const long long c0 = (long long)blockIdx.x << chunk_bits;
  const long long c1 = c0 + (1ll << chunk_bits) < count ? c0 + (1ll << chunk_bits) : count;
  double acc = 0.0;
  for (long long z = c0 + threadIdx.x; z < c1; z += blockDim.x) {
    const double pz = p[z];
    if (pz != 0.0) acc = fma(pz, cut_spin(n, As, half_total, (unsigned long long)z), acc);
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = part[0];
}

}  // namespace lrq

namespace lrq {
// element z <-> element 2^bits - 1 - z (the global bit flip X^(x)n on indices)
template <typename E>
__global__ void reverse_kernel(void* data, int bits) {
  E* a = reinterpret_cast<E*>(data);
  const long long N = 1ll << bits;
  const long long z = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (bits <= 0 || z >= N / 2) return;
  const E x = a[z];
  a[z] = a[N - 1 - z];
  a[N - 1 - z] = x;
}
}  // namespace lrq
