// Multi-GPU support (one process per GPU): NCCL loaded at run time, the
// per-rank phase terms of the distributed plan, and the global-qubit remap.
//
// Reference analog: lrqbench sharded.py:1-22,96-130,202-385 (threads holding
// 2^(nq-nq_local) shards that swap half-blocks per gate through queues).  Here
// every GPU holds 2^(n-g) amplitudes whose top g physical bits equal its rank;
// the cost phase needs no communication (the rank's qubits enter as a field
// and a constant), and the mixer of the g global qubits costs one all-to-all
// block transpose per layer instead of one pairwise exchange per gate.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>
#include <vector>

namespace lrq {

// NCCL entry points resolved with dlopen: the single-GPU engine never needs
// NCCL, and a process that already loaded torch's NCCL shares that copy.
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

inline NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      api.err = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
#define LRQ_NCCL_SYM(field, sym)                                       \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, #sym)); \
  if (!api.field) {                                                    \
    api.err = "NCCL symbol missing: " #sym;                            \
    return;                                                            \
  }
    LRQ_NCCL_SYM(GetUniqueId, ncclGetUniqueId)
    LRQ_NCCL_SYM(CommInitRank, ncclCommInitRank)
    LRQ_NCCL_SYM(CommDestroy, ncclCommDestroy)
    LRQ_NCCL_SYM(CommAbort, ncclCommAbort)
    LRQ_NCCL_SYM(Send, ncclSend)
    LRQ_NCCL_SYM(Recv, ncclRecv)
    LRQ_NCCL_SYM(GroupStart, ncclGroupStart)
    LRQ_NCCL_SYM(GroupEnd, ncclGroupEnd)
    LRQ_NCCL_SYM(AllGather, ncclAllGather)
    LRQ_NCCL_SYM(AllReduce, ncclAllReduce)
    LRQ_NCCL_SYM(GetErrorString, ncclGetErrorString)
    LRQ_NCCL_SYM(CommGetAsyncError, ncclCommGetAsyncError)
#undef LRQ_NCCL_SYM
    api.ok = true;
  });
  return api;
}

// physical bit -> logical qubit for permutation state `perm` (0: identity;
// 1: the g global bits [n_loc, n) swapped with the top local bits [n_loc-g, n_loc))
inline std::vector<int> dist_perm(int n, int g, int perm) {
  std::vector<int> pi(n);
  for (int k = 0; k < n; ++k) pi[k] = k;
  if (perm) {
    const int nl = n - g;
    for (int i = 0; i < g; ++i) {
      pi[nl - g + i] = nl + i;
      pi[nl + i] = nl - g + i;
    }
  }
  return pi;
}

// Local view of E_M(z) = sum_{i<j} M_ij s_i s_j on rank `rank`:
//   Mloc[a][b] = M[pi(a)][pi(b)]                     (local physical bits)
//   ext[a]     = sum_{j global} M[pi(a)][pi(j)] s_j  (field from the rank bits)
//   cst        = sum_{j<l global} M[pi(j)][pi(l)] s_j s_l
// with M given as n(n-1)/2 lexicographic edge values.
inline void dist_terms(int n, int g, int rank, int perm, const double* edges, double* Mloc, double* ext,
                       double* cst) {
  std::vector<double> M((size_t)n * n, 0.0);
  int e = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j, ++e) M[(size_t)i * n + j] = M[(size_t)j * n + i] = edges[e];
  const std::vector<int> pi = dist_perm(n, g, perm);
  const int nl = n - g;
  auto s = [&](int j) { return ((rank >> (j - nl)) & 1) ? -1.0 : 1.0; };
  for (int a = 0; a < nl; ++a) {
    for (int b = 0; b < nl; ++b) Mloc[(size_t)a * nl + b] = M[(size_t)pi[a] * n + pi[b]];
    double f = 0.0;
    for (int j = nl; j < n; ++j) f += M[(size_t)pi[a] * n + pi[j]] * s(j);
    ext[a] = f;
  }
  double c = 0.0;
  for (int j = nl; j < n; ++j)
    for (int l = j + 1; l < n; ++l) c += M[(size_t)pi[j] * n + pi[l]] * s(j) * s(l);
  *cst = c;
}

}  // namespace lrq
