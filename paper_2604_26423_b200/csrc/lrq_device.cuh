// Device-side building blocks for the LR-QAOA state-vector engine (sm_100a).
//
// Notation used throughout:
//   n      local qubits; amplitude index z has qubit k at bit k
//          (reference convention, lrqbench engine.py:3-4).
//   tile   2^K amplitudes handled by one CTA at a time.  Tile bit i maps to
//          global bit g(i) = i for i < m, q0 + (i - m) for i >= m, so every
//          tile is a union of 2^(K-m) contiguous runs of 2^m amplitudes.
//   layout "lo": each thread holds 2^RB amplitudes in registers whose tile
//          indices differ in tile bits [lo, lo+RB); the thread index fills the
//          other tile bits in ascending order.
//   E_M(z) = sum_{i<j} M_ij s_i s_j + sum_i ext_i s_i + cst,  s_k = 1 - 2 bit_k(z).
//          With M = J_k (per-layer RZZ half angles) exp(-i E_J) is the cost
//          phase of one layer; with M = w (edge weights) C(z) = (W - E_w)/2.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace lrq {

// Checked build (build.py --checked, -DLRQ_CHECKED -> _lib/liblrq_checked.so):
// device-side bounds and layout assertions in every kernel family; a failed
// check prints its line and traps (a launch error, not a silent corruption).
// The release build compiles them away.  This stands in for
// compute-sanitizer, which the GPU pool does not run.
#ifdef LRQ_CHECKED
#define LRQ_CHECK(cond)                                                                          \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("LRQ_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define LRQ_CHECK(cond) \
  do {                  \
  } while (0)
#endif
__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned v;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}
// the carved shared-memory layout ends inside the dynamic allocation
#define LRQ_CHECK_SMEM(base_raw, end_ptr) \
  LRQ_CHECK((size_t)((const unsigned char*)(end_ptr) - (const unsigned char*)(base_raw)) <= dyn_smem_bytes())

template <typename T> struct CxT;
template <> struct CxT<float> { typedef float2 V; };
template <> struct CxT<double> { typedef double2 V; };

__host__ __device__ constexpr int ctz_c(int k) { return (k & 1) ? 0 : 1 + ctz_c(k >> 1); }

__device__ __forceinline__ double spin(uint64_t z, int k) { return ((z >> k) & 1ull) ? -1.0 : 1.0; }

// ---------------------------------------------------------------------------
// complex helpers

__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(a), "f"(b));
  return u;
}
__device__ __forceinline__ float2 upk2(unsigned long long u) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(u));
  return r;
}
// packed a*b + c on two fp32 lanes (Blackwell FFMA2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)), "l"(pk2(c.x, c.y)));
  return upk2(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(r);
}

// x + i t y  (one half of the scaled RX butterfly)
__device__ __forceinline__ float2 bf_half(float2 x, float2 y, float2 tv /* (-t, t) */) {
#ifdef LRQ_EXPLICIT_FFMA2
  return ffma2(tv, make_float2(y.y, y.x), x);
#else
  return make_float2(fmaf(tv.x, y.y, x.x), fmaf(tv.y, y.x, x.y));
#endif
}
__device__ __forceinline__ double2 bf_half(double2 x, double2 y, double t) {
  return make_double2(fma(-t, y.y, x.x), fma(t, y.x, x.y));
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmul_conj(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cmul_amp(float2 a, double2 f) {
  float2 g = make_float2((float)f.x, (float)f.y);
  float2 m = fmul2(make_float2(a.y, a.y), make_float2(-g.y, g.x));
  return ffma2(make_float2(a.x, a.x), g, m);
}
__device__ __forceinline__ double2 cmul_amp(double2 a, double2 f) { return cmul(a, f); }

__device__ __forceinline__ double2 expmi(double angle) {  // exp(-i angle)
  double s, c;
  sincos(angle, &s, &c);
  return make_double2(c, -s);
}

// float32 phasor exp(-i angle) of a float64 angle: reduced mod 2pi in float64
// first (|angle| reaches ~1e2 rad), then an accurate float32 sincos
__device__ __forceinline__ float2 phasor32(double angle) {
  const double k = rint(angle * 0.15915494309189535);
  const float r = (float)fma(-k, 6.283185307179586, angle);
  float s, co;
  sincosf(r, &s, &co);
  return make_float2(co, -s);
}
#ifdef LRQ_EXPLICIT_FFMA2
// packed complex products: one FMUL2 + one FFMA2 (the broadcasts, lane swaps
// and one-lane negations are operand modifiers in SASS)
// a b = a.x b + a.y (i b),  i b = (-b.y, b.x)
__device__ __forceinline__ float2 cmul32(float2 a, float2 b) {
  return ffma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), fmul2(make_float2(a.x, a.x), b));
}
// a conj(b) = b.x a + b.y (-i a),  -i a = (a.y, -a.x)
__device__ __forceinline__ float2 cmul32_conj(float2 a, float2 b) {
  return ffma2(make_float2(b.y, b.y), make_float2(a.y, -a.x), fmul2(make_float2(b.x, b.x), a));
}
#else
__device__ __forceinline__ float2 cmul32(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmul32_conj(float2 a, float2 b) {  // a * conj(b)
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
#endif
__device__ __forceinline__ float2 conj32(float2 a) { return make_float2(a.x, -a.y); }

// ---------------------------------------------------------------------------
// streaming global access (each amplitude is read once and written once per
// sweep; the state is far larger than L2, so mark it evict-first)

// named barrier 1 over the 256 compute threads of a sweep CTA
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
// named barrier `id` over one 256-thread team
__device__ __forceinline__ void team_sync(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }
// named barrier `id` over `count` threads (a multiple of 32)
__device__ __forceinline__ void team_sync_n(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// ---- mbarrier / TMA primitives ---------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware (up to
// the hint, in ns) instead of spinning on issue slots the other warps need
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// bounded wait: a lost transaction traps (a recoverable launch error) after
// kMbarTrapNs of wall time instead of hanging the device.  The clock is read
// only once the fast path has failed, so a ready barrier costs one try_wait.
constexpr unsigned long long kMbarTrapNs = 20ull * 1000 * 1000 * 1000;  // 20 s
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  if (mbar_try_wait(b, parity)) return;
  const unsigned long long t0 = global_ns();
  while (!mbar_try_wait(b, parity))
    if (global_ns() - t0 > kMbarTrapNs) __trap();
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const void* tmap, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const void* tmap, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_5d(const void* tmap, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most N committed bulk groups still read shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// TMA tensor prefetch of one 5-D box into L2
__device__ __forceinline__ void tma_prefetch_5d(const void* tmap, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
// TMA bulk prefetch of [p, p+bytes) into L2 (bytes: multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ float4 ld_unit(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_unit(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ void st_unit(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_unit(double2* p, double2 v) { __stcs(p, v); }

// |a|^2 in float64 with the reference's rounding: re*re and im*im each rounded,
// then added (engine.py:94-96) — no FMA contraction.
// complex64: both squares are exact in fp64 (24-bit mantissas), so one
// rounding of x^2 + y^2 (the fma) equals the reference's float64 re^2 + im^2
__device__ __forceinline__ double prob(float2 a) {
  double x = (double)a.x, y = (double)a.y;
  return __fma_rn(x, x, __dmul_rn(y, y));
}
__device__ __forceinline__ double prob(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

// p-weighted energy histogram bin update (SweepParams::hist): fixed point
// with 2^60 per unit probability, integer atomics (order-independent sums)
constexpr double kHistOne = 1152921504606846976.0;  // 2^60: fixed-point unit of a histogram bin
__device__ __forceinline__ void hist_add(unsigned long long* h, int bins, double lo, double scale, double e,
                                         double p) {
  int b = (int)floor((e - lo) * scale);
  b = b < 0 ? 0 : (b >= bins ? bins - 1 : b);
  const unsigned long long q = (unsigned long long)__double2ll_rn(p * kHistOne);
  if (q) atomicAdd(h + b, q);
}

}  // namespace lrq
