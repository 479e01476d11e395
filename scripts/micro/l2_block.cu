// Microbenchmark (not product code): can consecutive sweeps that only touch
// the low 22-23 bits of the index run out of L2?  Between two sweeps of the
// top group, the sweeps M(A), F(H), M(A) of an n=32 complex64 plan never mix
// index bits >= 23, so they can run super-block by super-block (2^23
// amplitudes = 64 MB), each super-block's three passes back to back while it
// sits in the 126 MB L2, DRAM seeing one round trip instead of three.
//
// Memory-only model: a "tile pass" loads a 64 KB tile's 16-byte units
// (pattern A: contiguous; H: 64 B runs, 10 targets at 2^13; H4: 128 B runs,
// 9 targets at 2^13), perturbs them and stores them back.  Modes:
//   full X         one pass of pattern X over the whole state (DRAM bound)
//   block X,Y,Z    per super-block: pass X, grid barrier, pass Y, barrier,
//                  pass Z, barrier (one persistent kernel)
// Prints ms and the equivalent GB/s (passes * 2 * state bytes / time).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_block l2_block.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

struct Pat {
  int run_u_bits, k, q0_u_bits;  // run of 2^run units, k targets at unit bit q0
};
// 16-byte units: a 64 KB tile is 4096 units (12 bits)
static const Pat PA = {12, 0, 12}, PH = {2, 10, 12}, PH4 = {3, 9, 12};

__device__ __forceinline__ long long unit_addr(const Pat& p, long long t, long long e) {
  const long long mid_count = 1ll << (p.q0_u_bits - p.run_u_bits);
  const long long mid = t & (mid_count - 1), outer = t >> (p.q0_u_bits - p.run_u_bits);
  const long long base = (outer << (p.q0_u_bits + p.k)) + (mid << p.run_u_bits);
  const long long j = e >> p.run_u_bits, o = e & ((1ll << p.run_u_bits) - 1);
  return base + (j << p.q0_u_bits) + o;
}

constexpr int U = 8;  // units per thread per chunk
constexpr int TPB = 256;
constexpr int CHUNK_BITS = 11;  // 8 * 256 = 2048 units per chunk (half a tile)

template <int HINT>
__device__ __forceinline__ void touch_chunk(uint4* a, const Pat& p, long long chunk) {
  const long long t = chunk >> 1;
  const long long e0 = (chunk & 1) << CHUNK_BITS;
  uint4 r[U];
  long long ad[U];
#pragma unroll
  for (int i = 0; i < U; ++i) {
    ad[i] = unit_addr(p, t, e0 + i * TPB + threadIdx.x);
    if (HINT == 1) r[i] = __ldcs(a + ad[i]);
    else r[i] = a[ad[i]];
  }
#pragma unroll
  for (int i = 0; i < U; ++i) {
    r[i].x ^= 1u;
    if (HINT == 1) __stcs(a + ad[i], r[i]);
    else a[ad[i]] = r[i];
  }
}

template <int HINT>
__global__ void __launch_bounds__(TPB) full_pass(uint4* a, Pat p, long long chunks) {
  for (long long c = blockIdx.x; c < chunks; c += gridDim.x) touch_chunk<HINT>(a, p, c);
}

__device__ unsigned g_count;
__device__ volatile unsigned g_gen;

__device__ __forceinline__ void grid_barrier(unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nblocks - 1) {
      g_count = 0;
      __threadfence();
      g_gen = gen + 1;
    } else {
      while (g_gen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// per super-block: the three passes, barriers between them; tiles of a
// super-block are the contiguous tile range [b * tpb, (b + 1) * tpb) for
// every pattern (the super-block is bits 0 .. q0 + k of the unit index)
__global__ void __launch_bounds__(TPB) block_passes(uint4* a, Pat p0, Pat p1, Pat p2, long long blocks,
                                                    long long tiles_per_block, int npass) {
  const Pat ps[3] = {p0, p1, p2};
  const long long cpb = tiles_per_block * 2;
  for (long long b = 0; b < blocks; ++b) {
    for (int s = 0; s < npass; ++s) {
      for (long long c = blockIdx.x; c < cpb; c += gridDim.x) touch_chunk<0>(a, ps[s], b * cpb + c);
      grid_barrier(gridDim.x);
    }
  }
}

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                              \
    }                                                                       \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32;  // complex64 amplitudes
  const long long units = 1ll << (n - 1);
  const size_t bytes = (size_t)units * 16;
  uint4* a;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMemset(a, 0, bytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_passes, TPB, 0));
  if (per_sm > 4) per_sm = 4;
  const long long tiles = units >> 12, chunks = tiles * 2;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto time_it = [&](auto fn) {
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      CK(cudaEventRecord(e0));
      fn();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
    return best;
  };
  printf("# l2_block n=%d complex64 (%.1f GiB), %d SMs, %d CTAs/SM x %d threads; GB/s = passes*2*state/time\n", n,
         bytes / 1073741824.0, sms, per_sm, TPB);
  struct {
    const char* name;
    Pat p;
  } pats[3] = {{"A", PA}, {"H(64B,q13)", PH}, {"H4(128B,q13)", PH4}};
  for (int i = 0; i < 3; ++i)
    for (int hint = 0; hint < 2; ++hint) {
      const Pat p = pats[i].p;
      const int grid = sms * per_sm;
      float ms = time_it([&] {
        if (hint) full_pass<1><<<grid, TPB>>>(a, p, chunks);
        else full_pass<0><<<grid, TPB>>>(a, p, chunks);
      });
      printf("full  %-14s %-8s %9.3f ms %8.1f GB/s\n", pats[i].name, hint ? "stream" : "default", ms,
             2.0 * bytes / (ms * 1e6));
    }
  struct {
    const char* name;
    Pat p0, p1, p2;
    int npass, sb;  // super-block: 2^sb units
  } combos[] = {{"A,H,A", PA, PH, PA, 3, 22},  {"A,H", PA, PH, PA, 2, 22},   {"A,H4,A", PA, PH4, PA, 3, 21},
                {"H,H,H", PH, PH, PH, 3, 22},  {"A,A,A", PA, PA, PA, 3, 22}, {"A,A,A", PA, PA, PA, 3, 20},
                {"A,A,A", PA, PA, PA, 3, 18},  {"A", PA, PA, PA, 1, 22},     {"H", PH, PH, PH, 1, 22}};
  for (auto& c : combos) {
    const long long tpb = 1ll << (c.sb - 12), blocks = tiles / tpb;
    const int grid = sms * per_sm;
    float ms = time_it([&] { block_passes<<<grid, TPB>>>(a, c.p0, c.p1, c.p2, blocks, tpb, c.npass); });
    printf("block %-14s sb=%3lld MB %9.3f ms %8.1f GB/s  (%.3f ms per pass)\n", c.name, (16ll << c.sb) >> 20, ms,
           c.npass * 2.0 * bytes / (ms * 1e6), ms / c.npass);
  }
  CK(cudaFree(a));
  return 0;
}
