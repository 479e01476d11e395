// Microbenchmark (not product code): pure TMA copy of a state in the sweep
// tile shapes, no compute.  One persistent CTA per SM, one thread drives a
// ring of NST 64 KB stages: load tile -> (wait) -> store -> (wait read) ->
// reload.  Reports GB/s (read + write) for the contiguous A tile (3-D box)
// and the strided high-group tiles (5-D box, 64 / 128 / 256 B runs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_copy tma_copy.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int NST, int SB>
__global__ void __launch_bounds__(32, 1) copy_kernel(const __grid_constant__ CUtensorMap tm, long long tiles, int bl,
                                                     int dims, int h3) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* st = sm + ((1024 - (su(sm) & 1023)) & 1023);
  __shared__ uint64_t bar[NST];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  auto load = [&](int s, long long tid) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(SB));
    const int c3 = h3 ? (int)(tid & 1) * h3 : 0;
    if (h3) tid >>= 1;
    if (dims == 3) {
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
              su(st + s * SB)),
          "l"(&tm), "r"(0), "r"(0), "r"((int)(2 * tid)), "r"(su(&bar[s]))
          : "memory");
    } else {
      const int c1 = (int)(tid & ((1ll << bl) - 1)), c4 = (int)(tid >> bl);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
              su(st + s * SB)),
          "l"(&tm), "r"(0), "r"(0), "r"(c1), "r"(c3), "r"(c4), "r"(su(&bar[s]))
          : "memory");
    }
  };
  auto store = [&](int s, long long tid) {
    const int c3 = h3 ? (int)(tid & 1) * h3 : 0;
    if (h3) tid >>= 1;
    if (dims == 3) {
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tm),
                   "r"(0), "r"(0), "r"((int)(2 * tid)), "r"(su(st + s * SB))
                   : "memory");
    } else {
      const int c1 = (int)(tid & ((1ll << bl) - 1)), c4 = (int)(tid >> bl);
      asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(&tm),
                   "r"(0), "r"(0), "r"(c1), "r"(c3), "r"(c4), "r"(su(st + s * SB))
                   : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  for (int s = 0; s < NST; ++s) {
    const long long tid = blockIdx.x + (long long)s * gridDim.x;
    if (tid < tiles) load(s, tid);
  }
  for (long long k = 0;; ++k) {
    const long long tid = blockIdx.x + k * gridDim.x;
    if (tid >= tiles) break;
    const int s = (int)(k % NST);
    const unsigned par = (unsigned)((k / NST) & 1);
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(su(&bar[s])),
        "r"(par)
        : "memory");
    store(s, tid);
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    const long long nxt = blockIdx.x + (k + NST) * gridDim.x;
    if (nxt < tiles) load(s, nxt);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// variant: TMA tensor load, then the CTA's 128 threads read the stage in
// memory order and write it back with coalesced 16-byte stores (no TMA store)
template <int NST>
__global__ void __launch_bounds__(128, 1) copy_stg_kernel(const __grid_constant__ CUtensorMap tm, long long tiles,
                                                          int bl, int MU, int qU, float4* amps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* st = sm + ((1024 - (su(sm) & 1023)) & 1023);
  __shared__ uint64_t bar[NST];
  const int t = threadIdx.x;
  if (t == 0) {
    for (int s = 0; s < NST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto load = [&](int s, long long tid) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(65536));
    const int c1 = (int)(tid & ((1ll << bl) - 1)), c4 = (int)(tid >> bl);
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            su(st + s * 65536)),
        "l"(&tm), "r"(0), "r"(0), "r"(c1), "r"(0), "r"(c4), "r"(su(&bar[s]))
        : "memory");
  };
  if (t == 0)
    for (int s = 0; s < NST; ++s) {
      const long long tid = blockIdx.x + (long long)s * gridDim.x;
      if (tid < tiles) load(s, tid);
    }
  const int swm = MU == 2 ? 3 : 7;
  for (long long k = 0;; ++k) {
    const long long tid = blockIdx.x + k * gridDim.x;
    if (tid >= tiles) break;
    const int s = (int)(k % NST);
    const unsigned par = (unsigned)((k / NST) & 1);
    asm volatile(
        "{ .reg .pred p; W2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W2; }" ::"r"(su(&bar[s])),
        "r"(par)
        : "memory");
    const uint64_t ut = (uint64_t)tid;
    const uint64_t baseU = ((ut & ((1ull << bl) - 1ull)) << MU) | ((ut >> bl) << (qU + 12 - MU));
    const float4* sv = reinterpret_cast<const float4*>(st + s * 65536);
    float4 r[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = j * 128 + t;
      r[j] = sv[e ^ ((e >> 3) & swm)];
    }
    __syncthreads();
    if (t == 0) {
      const long long nxt = blockIdx.x + (k + NST) * gridDim.x;
      if (nxt < tiles) load(s, nxt);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int e = j * 128 + t;
      const uint64_t g = baseU + (uint64_t)(e & ((1 << MU) - 1)) + ((uint64_t)(e >> MU) << qU);
      __stcs(amps + g, r[j]);
    }
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 30;  // complex64 amplitudes: 8 GiB
  const size_t bytes = (size_t)8 << n;
  void* a = nullptr;
  cudaMalloc(&a, bytes);
  cudaMemset(a, 0, bytes);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long tiles = 1ll << (n - 13);
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  struct Case { const char* name; int MA; int q0; };
  // MA = run amp bits (3: 64 B, 4: 128 B, 5: 256 B); q0 = first group qubit
  Case cases[] = {{"A contiguous 64 KB", 0, 0}, {"H 64 B runs q0=13", 3, 13}, {"H4 128 B runs q0=21", 4, 21},
                  {"H4 128 B runs q0=13", 4, 13}, {"H 64 B runs q0=21", 3, 21}};
  for (const Case& c : cases) {
    CUtensorMap tm;
    int dims = 3, bl = 0;
    CUresult r;
    if (c.MA == 0) {
      cuuint64_t d[3] = {16, 256, 2ull * tiles};
      cuuint64_t str[2] = {128, 32768};
      cuuint32_t box[3] = {16, 256, 2};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, a, d, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      dims = 5;
      const int KA = 13, nrb = KA - c.MA, q0 = c.q0;
      cuuint64_t d[5] = {1ull << c.MA, 32, 1ull << (q0 - c.MA), 1ull << (nrb - 5), 1ull << (n - q0 - nrb)};
      cuuint64_t str[4] = {(1ull << q0) * 8, (1ull << c.MA) * 8, (1ull << (q0 + 5)) * 8, (1ull << (q0 + nrb)) * 8};
      cuuint32_t box[5] = {(cuuint32_t)(1u << c.MA), 32, 1, (cuuint32_t)(1u << (nrb - 5)), 1};
      r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, d, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              c.MA == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      bl = q0 - c.MA;
    }
    if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, (int)r); continue; }
    const size_t smem = 3 * 65536 + 1024;
    cudaFuncSetAttribute(copy_kernel<3, 65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      copy_kernel<3, 65536><<<sms, 32, smem>>>(tm, tiles, bl, dims, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-22s TMA ld+st   %7.3f ms  %7.1f GB/s (read+write)  %s\n", c.name, best, 2.0 * bytes / (best * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    if (dims == 5) {
      // deeper ring: half-tile boxes (32 KB) in 6 stages
      const int KA = 13, nrb = KA - c.MA, q0 = c.q0;
      cuuint64_t d[5] = {1ull << c.MA, 32, 1ull << (q0 - c.MA), 1ull << (nrb - 5), 1ull << (n - q0 - nrb)};
      cuuint64_t str[4] = {(1ull << q0) * 8, (1ull << c.MA) * 8, (1ull << (q0 + 5)) * 8, (1ull << (q0 + nrb)) * 8};
      const cuuint32_t half = (cuuint32_t)(1u << (nrb - 5)) / 2;
      cuuint32_t box[5] = {(cuuint32_t)(1u << c.MA), 32, 1, half, 1};
      CUtensorMap th;
      enc(&th, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, a, d, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          c.MA == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      cudaFuncSetAttribute(copy_kernel<6, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      best = 1e9f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        copy_kernel<6, 32768><<<sms, 32, smem>>>(th, 2 * tiles, bl, dims, (int)half);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      err = cudaGetLastError();
      printf("%-22s TMA 6x32KB  %7.3f ms  %7.1f GB/s (read+write)  %s\n", c.name, best,
             2.0 * bytes / (best * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
      cudaFuncSetAttribute(copy_stg_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      best = 1e9f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        copy_stg_kernel<3><<<sms, 128, smem>>>(tm, tiles, bl, c.MA - 1, c.q0 - 1, (float4*)a);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
      }
      err = cudaGetLastError();
      printf("%-22s TMA ld+STG  %7.3f ms  %7.1f GB/s (read+write)  %s\n", c.name, best,
             2.0 * bytes / (best * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  }
  return 0;
}
