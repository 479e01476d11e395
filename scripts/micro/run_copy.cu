// Microbenchmark (not product code): the DRAM ceiling of the access patterns
// a mixer sweep can use.  A state of 2^n 8-byte units (complex64 amplitudes)
// is copied in place, tile by tile; a tile is 2^k runs of `run` contiguous
// bytes, the runs 2^q0 units apart (q0 = the first target qubit of the
// group), exactly the shape of a high-group sweep tile with k targets.
// Two engines: plain 16-byte LDG/STG from registers (LSU path) and a TMA
// 3-D box ring (one thread, 3 stages).  Prints GB/s counted as read+write.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o run_copy run_copy.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// LSU copy: each CTA (256 threads) takes whole tiles; per round every thread
// holds U 16-byte units (U*256*16 bytes in flight per CTA)
template <int U>
__global__ void __launch_bounds__(256) lsu_copy(uint4* __restrict__ a, long long tiles, int run_u_bits, int k,
                                                int q0_u_bits, long long mid_count, int tile_u_bits) {
  const long long chunks_per_tile = 1ll << (tile_u_bits - 8 - __builtin_ctz(U));
  const long long total = tiles * chunks_per_tile;
  for (long long c = blockIdx.x; c < total; c += gridDim.x) {
    const long long t = c / chunks_per_tile, part = c % chunks_per_tile;
    const long long mid = t % mid_count, outer = t / mid_count;
    const long long base = (outer << (q0_u_bits + k)) + (mid << run_u_bits);
    uint4 r[U];
    long long addr[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const long long e = ((part * U + i) << 8) + threadIdx.x;  // unit index inside the tile
      const long long j = e >> run_u_bits, o = e & ((1ll << run_u_bits) - 1);
      addr[i] = base + (j << q0_u_bits) + o;
      r[i] = __ldcs(a + addr[i]);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) __stcs(a + addr[i], r[i]);
  }
}

// out-of-place LSU copy: one side uses the strided tile pattern, the other
// writes/reads the tile as one contiguous block (mode 0: strided read ->
// contiguous write; mode 1: contiguous read -> strided write)
template <int U>
__global__ void __launch_bounds__(256) lsu_oop(const uint4* __restrict__ src, uint4* __restrict__ dst, long long tiles,
                                               int run_u_bits, int k, int q0_u_bits, long long mid_count,
                                               int tile_u_bits, int mode) {
  const long long chunks_per_tile = 1ll << (tile_u_bits - 8 - __builtin_ctz(U));
  const long long total = tiles * chunks_per_tile;
  for (long long c = blockIdx.x; c < total; c += gridDim.x) {
    const long long t = c / chunks_per_tile, part = c % chunks_per_tile;
    const long long mid = t % mid_count, outer = t / mid_count;
    const long long base = (outer << (q0_u_bits + k)) + (mid << run_u_bits);
    uint4 r[U];
    long long sa[U], ca[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const long long e = ((part * U + i) << 8) + threadIdx.x;
      const long long j = e >> run_u_bits, o = e & ((1ll << run_u_bits) - 1);
      sa[i] = base + (j << q0_u_bits) + o;
      ca[i] = (t << tile_u_bits) + e;
      r[i] = __ldcs(src + (mode == 0 ? sa[i] : ca[i]));
    }
#pragma unroll
    for (int i = 0; i < U; ++i) __stcs(dst + (mode == 0 ? ca[i] : sa[i]), r[i]);
  }
}

// TMA copy: 5-D box {run elems, 1 mid, 2^k1, 2^k2 runs, 1} over dims {run, mid,
// 2^k1, 2^k2 (stride 2^q0), rest}.  G > 1: a CTA copies G adjacent tiles (mid
// index m..m+G-1, i.e. G adjacent runs) back to back and, when it starts a
// group, prefetches its next group into L2 with one tensor prefetch through
// pm, whose box has G-times longer runs (the DRAM then sees G*run bytes).
__device__ __forceinline__ void tma_pf5(const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4) {
  asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(m), "r"(c0), "r"(c1),
               "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
template <int NST>
__global__ void __launch_bounds__(32, 1) tma_copy(const __grid_constant__ CUtensorMap tm,
                                                  const __grid_constant__ CUtensorMap pm, long long tiles,
                                                  long long mid_count, int sb, int G) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* st = sm + ((1024 - (su(sm) & 1023)) & 1023);
  __shared__ uint64_t bar[NST];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  // k-th tile of this CTA
  auto tile_of = [&](long long k) -> long long {
    return (blockIdx.x + (k / G) * (long long)gridDim.x) * G + (k % G);
  };
  auto coords = [&](long long tid, int& c0, int& c2) {
    c0 = (int)(tid % mid_count);
    c2 = (int)(tid / mid_count);
  };
  auto load = [&](int s, long long tid) {
    int c0, c2;
    coords(tid, c0, c2);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(sb));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su(st + s * sb)),
        "l"(&tm), "r"(0), "r"(c0), "r"(0), "r"(0), "r"(c2), "r"(su(&bar[s]))
        : "memory");
  };
  auto store = [&](int s, long long tid) {
    int c0, c2;
    coords(tid, c0, c2);
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&tm),
                 "r"(0), "r"(c0), "r"(0), "r"(0), "r"(c2), "r"(su(st + s * sb))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  auto prefetch_group = [&](long long first_tile) {
    if (G <= 1 || first_tile >= tiles) return;
    int c0, c2;
    coords(first_tile, c0, c2);
    tma_pf5(&pm, 0, c0 / G, 0, 0, c2);
  };
  if (G > 1) {
    prefetch_group(tile_of(0));
    prefetch_group(tile_of(G));
  }
  for (int s = 0; s < NST; ++s) {
    const long long tid = tile_of(s);
    if (tid < tiles) load(s, tid);
  }
  for (long long k = 0;; ++k) {
    const long long tid = tile_of(k);
    if (tid >= tiles) break;
    const int s = (int)(k % NST);
    const unsigned par = (unsigned)((k / NST) & 1);
    if (G > 1 && k % G == 0) prefetch_group(tile_of(k + 2 * G));
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su(&bar[s])),
        "r"(par)
        : "memory");
    store(s, tid);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    const long long nxt = tile_of(k + NST);
    if (nxt < tiles) load(s, nxt);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float time_it(void (*fn)(void*), void* ctx) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    fn(ctx);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

struct Ctx {
  uint4* a;
  long long tiles, mid;
  int run_u_bits, k, q0_u_bits, tile_u_bits, grid, ctas_per_sm;
  uint4* b;
  int mode;
  CUtensorMap tm, pm;
  int sb, G;
};

template <int U>
static void run_lsu(void* p) {
  Ctx* c = (Ctx*)p;
  lsu_copy<U><<<c->grid, 256>>>(c->a, c->tiles, c->run_u_bits, c->k, c->q0_u_bits, c->mid, c->tile_u_bits);
}
static void run_oop(void* p) {
  Ctx* c = (Ctx*)p;
  lsu_oop<16><<<c->grid, 256>>>(c->a, c->b, c->tiles, c->run_u_bits, c->k, c->q0_u_bits, c->mid, c->tile_u_bits,
                                c->mode);
}
static void run_tma(void* p) {
  Ctx* c = (Ctx*)p;
  tma_copy<3><<<c->grid, 32, 3 * c->sb + 1024>>>(c->tm, c->pm, c->tiles, c->mid, c->sb, c->G);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32;  // 8-byte units: 2^n * 8 bytes
  const size_t bytes = (size_t)8 << n;
  void* a = nullptr;
  if (cudaMalloc(&a, bytes) != cudaSuccess) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 0, bytes);
  void* b2 = nullptr;
  if (cudaMalloc(&b2, bytes) != cudaSuccess) b2 = nullptr;
  if (b2) cudaMemset(b2, 0, bytes);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_copy<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536 + 1024);
  printf("# run_copy n=%d (%zu GiB, 8-byte units), %d SMs; GB/s = 2*bytes/time (read+write), best of 3\n", n,
         bytes >> 30, sms);
  printf("%-6s %-6s %-4s %-10s %10s %10s %10s %10s %10s %10s %10s\n", "run_B", "tileKB", "q0", "stride_B", "LSU_U8", "LSU_U16",
         "TMA", "TMA_G2pf", "TMA_G4pf", "OOP_rdS", "OOP_wrS");
  struct Case { int rb, q0, tk; };
  const Case cases[] = {{64, 13, 64}, {64, 22, 64}, {128, 13, 64}, {128, 23, 64}, {256, 13, 64}, {256, 22, 64},
                        {512, 22, 64}, {64, 13, 32}, {128, 23, 32}, {256, 22, 32}};
  for (const Case& cs : cases) {
    const int rb = cs.rb, q0 = cs.q0, tile_b = cs.tk * 1024;
    const int run_u = __builtin_ctz(rb / 8);
    const int k = __builtin_ctz(tile_b / rb);
    if (q0 + k > n) continue;
    Ctx c;
    c.a = (uint4*)a;
    c.run_u_bits = run_u - 1;
    c.k = k;
    c.q0_u_bits = q0 - 1;
    c.tile_u_bits = __builtin_ctz(tile_b / 16);
    c.mid = (1ll << (q0 - run_u));
    c.tiles = (long long)(bytes / tile_b);
    c.grid = sms * 4;
    float l8 = time_it(run_lsu<8>, &c);
    float l16 = c.tile_u_bits >= 12 ? time_it(run_lsu<16>, &c) : -1.f;
    float tg[3] = {-1.f, -1.f, -1.f};
    const int k1 = k < 8 ? k : 8, k2 = k - k1;
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    for (int gi = 0; gi < 3; ++gi) {
      const int G = 1 << gi;
      if (G * rb > 2048 || c.mid % G) continue;
      cuuint64_t d[5] = {(cuuint64_t)(rb / 8), (cuuint64_t)c.mid, (cuuint64_t)(1ull << k1), (cuuint64_t)(1ull << k2),
                         (cuuint64_t)(1ull << (n - q0 - k))};
      cuuint64_t str[4] = {(cuuint64_t)rb, (1ull << q0) * 8, (1ull << (q0 + k1)) * 8, (1ull << (q0 + k)) * 8};
      cuuint32_t box[5] = {(cuuint32_t)(rb / 8), 1, (cuuint32_t)(1u << k1), (cuuint32_t)(1u << k2), 1};
      cuuint64_t dp[5] = {(cuuint64_t)(G * rb / 8), (cuuint64_t)(c.mid / G), (cuuint64_t)(1ull << k1),
                          (cuuint64_t)(1ull << k2), (cuuint64_t)(1ull << (n - q0 - k))};
      cuuint64_t sp[4] = {(cuuint64_t)(G * rb), (1ull << q0) * 8, (1ull << (q0 + k1)) * 8, (1ull << (q0 + k)) * 8};
      cuuint32_t bp[5] = {(cuuint32_t)(G * rb / 8), 1, (cuuint32_t)(1u << k1), (cuuint32_t)(1u << k2), 1};
      if (k2 > 8) continue;
      if (enc(&c.tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, d, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        continue;
      if (enc(&c.pm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, dp, sp, bp, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        continue;
      c.sb = tile_b;
      c.G = G;
      c.grid = sms;
      tg[gi] = time_it(run_tma, &c);
    }
    float oo[2] = {-1.f, -1.f};
    if (b2 && c.tile_u_bits >= 12) {
      c.b = (uint4*)b2;
      c.grid = sms * 4;
      for (int m = 0; m < 2; ++m) {
        c.mode = m;
        oo[m] = time_it(run_oop, &c);
      }
    }
    cudaError_t err = cudaGetLastError();
    auto gbs = [&](float ms) { return ms > 0 ? 2.0 * bytes / (ms * 1e-3) / 1e9 : 0.0; };
    printf("%-6d %-6d %-4d %-10lld %10.1f %10.1f %10.1f %10.1f %10.1f %10.1f %10.1f %s\n", rb, cs.tk, q0,
           (long long)(8ll << q0), gbs(l8), gbs(l16), gbs(tg[0]), gbs(tg[1]), gbs(tg[2]), gbs(oo[0]), gbs(oo[1]),
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    fflush(stdout);
  }
  return 0;
}
