// Microbenchmark (not product code): TMA copy / store-only of 64 KB tiles of
// 2^9 runs x 256 B (complex64 group C9 at q0 = 23, n = 32) with the box
// forms and tile orders the cluster sweep uses, against the 128 B-run H4
// tile of the single-CTA sweep.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o box_copy box_copy.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// order 0: tile k of CTA b = b + k*grid; order 1: cluster pairs - CTA b takes
// half (b & 1) of pair (b >> 1) + k*(grid/2), the half bit being the lowest
// tile-index bit above `bl` low bits
template <int NST>
__global__ void __launch_bounds__(32, 1) tma_tiles(const __grid_constant__ CUtensorMap tm, long long tiles, int bl,
                                                   int order, int store_only) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* st = sm + ((1024 - (su(sm) & 1023)) & 1023);
  __shared__ uint64_t bar[NST];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto tile_of = [&](long long k) -> long long {
    if (order == 0) return blockIdx.x + k * (long long)gridDim.x;
    const long long pt = (blockIdx.x >> 1) + k * (long long)(gridDim.x >> 1);
    if (pt >= tiles / 2) return tiles;
    return ((((pt >> bl) << 1) | (blockIdx.x & 1)) << bl) | (pt & ((1ll << bl) - 1));
  };
  auto load = [&](int s, long long tid) {
    const int c1 = (int)(tid & ((1ll << bl) - 1)), c4 = (int)(tid >> bl);
    if (store_only) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar[s])));
      return;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(65536));
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(su(st + s * 65536)),
        "l"(&tm), "r"(0), "r"(0), "r"(c1), "r"(0), "r"(c4), "r"(su(&bar[s]))
        : "memory");
  };
  auto store = [&](int s, long long tid) {
    const int c1 = (int)(tid & ((1ll << bl) - 1)), c4 = (int)(tid >> bl);
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&tm),
                 "r"(0), "r"(0), "r"(c1), "r"(0), "r"(c4), "r"(su(st + s * 65536))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  for (int s = 0; s < NST; ++s) {
    const long long tid = tile_of(s);
    if (tid < tiles) load(s, tid);
  }
  for (long long k = 0;; ++k) {
    const long long tid = tile_of(k);
    if (tid >= tiles) break;
    const int s = (int)(k % NST);
    const unsigned par = (unsigned)((k / NST) & 1);
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

int main() {
  const int n = 32;
  const size_t bytes = (size_t)8 << n;
  void* a = nullptr;
  if (cudaMalloc(&a, bytes) != cudaSuccess) return 1;
  cudaMemset(a, 0, bytes);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_tiles<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536 + 1024);
  const long long tiles = 1ll << (n - 13);
  struct Case { const char* name; int MA, q0, form; };  // form 0: {16, 32, 1, 2^(nrb-5), 1} (H-style); 1: {16, 2^(MA-4), 1, 2^nrb, 1}
  Case cases[] = {{"H4 128B q0=23 (sweep now)", 4, 23, 0}, {"C9 256B q0=23 {16,2,..,256} sw128", 5, 23, 1},
                  {"C10 128B q0=13 {16,32,..,16}", 4, 13, 0}, {"H 64B q0=13", 3, 13, 2}};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  printf("# box_copy n=32 c64 (32 GiB): GB/s (copy: read+write; store-only: write)\n");
  for (const Case& c : cases) {
    const int nrb = 13 - c.MA, q0 = c.q0;
    CUtensorMap tm;
    CUresult r;
    if (c.form == 1) {
      cuuint64_t d[5] = {16, 1ull << (c.MA - 4), 1ull << (q0 - c.MA), 1ull << nrb, 1ull << (n - q0 - nrb)};
      cuuint64_t str[4] = {128, (1ull << c.MA) * 8, (1ull << q0) * 8, (1ull << (q0 + nrb)) * 8};
      cuuint32_t box[5] = {16, (cuuint32_t)(1u << (c.MA - 4)), 1, (cuuint32_t)(1u << nrb), 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, d, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      cuuint64_t d[5] = {1ull << c.MA, 32, 1ull << (q0 - c.MA), 1ull << (nrb - 5), 1ull << (n - q0 - nrb)};
      cuuint64_t str[4] = {(1ull << q0) * 8, (1ull << c.MA) * 8, (1ull << (q0 + 5)) * 8, (1ull << (q0 + nrb)) * 8};
      cuuint32_t box[5] = {(cuuint32_t)(1u << c.MA), 32, 1, (cuuint32_t)(1u << (nrb - 5)), 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, d, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              c.MA == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", c.name, (int)r);
      continue;
    }
    const int bl = q0 - c.MA;
    for (int so = 0; so < 2; ++so)
      for (int order = 0; order < 2; ++order) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9f;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          tma_tiles<3><<<sms, 32, 3 * 65536 + 1024>>>(tm, tiles, bl, order, so);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          if (rep && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        printf("%-40s %-10s %-11s %8.3f ms %8.1f GB/s %s\n", c.name, so ? "store-only" : "copy",
               order ? "pair-split" : "consecutive", best, (so ? 1.0 : 2.0) * bytes / (best * 1e-3) / 1e9,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
      }
  }
  return 0;
}
