// liblrq.so — host engine and C ABI (include/lrq.h) for the B200-native
// LR-QAOA state-vector path.  Replaces lrqbench engine.py:198-273 and
// problem.py:139-211 behind the reference's own entry points (the Python
// mirror in paper_2604_26423_b200 calls these through ctypes).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing without a profiler attached

#include "../../include/lrq.h"
#include "lrq_aux.cuh"
#include "lrq_plan.h"
#include "lrq_dist.cuh"
#include "lrq_sweep_tma.cuh"
#include "lrq_sweep_wd.cuh"
#include "lrq_sweep_wdc.cuh"

using namespace lrq;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? LRQ_ECAPACITY : LRQ_ERUNTIME,             \
                  std::string("CUDA error in ") + #expr + ": " + cudaGetErrorString(e_));    \
    }                                                                                         \
  } while (0)

// per-tile reduction arrays (sum p, sum pE, min E, argmin, max E), finalize
// outputs (the same five scalars) and the multi-CTA finalize scratch
constexpr int kRedArrays = 5;
constexpr int kOutScalars = 5;
constexpr int kFinScratch = 6 * kFinBlocks;

// tile geometry: 4096 16-byte units per tile = 2^(12+pair)
// amplitudes (pair = 1 for complex64: a unit holds two amplitudes)
inline int pair_of(int pbytes) { return pbytes == 8 ? 1 : 0; }
inline int tile_amp_bits(int pbytes) { return kUnitBits + pair_of(pbytes); }

// NVTX range over a host scope (nsys / ncu --nvtx show the engine's phases:
// runs, sweeps by kind and group, remaps, sampling)
struct NvtxRange {
  explicit NvtxRange(const char* msg) { nvtxRangePushA(msg); }
  NvtxRange(const char* a, const char* b) {
    char buf[96];
    snprintf(buf, sizeof buf, "%s%s", a, b);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
const char* group_name(int gk) {
  return gk == GK_A ? "(A)" : gk == GK_H4 ? "(H4)" : gk == GK_C10 ? "(C10)" : gk == GK_C9 ? "(C9)" : gk == GK_C8 ? "(C8)" : "(H)";
}

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

template <typename T, int GK, int SK>
int launch_sweep_t(cudaStream_t st, const SweepParams& sp, int grid, size_t smem) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(sweep_kernel<T, GK, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  CUDA_TRY(err);
  sweep_kernel<T, GK, SK><<<grid, kThreads, smem, st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  return LRQ_OK;
}

template <typename T>
int launch_sweep_kind(cudaStream_t st, int gk, int sk, const SweepParams& sp, int grid, size_t smem) {
  if (gk == GK_A) {
    switch (sk) {
      case SK_P: return launch_sweep_t<T, GK_A, SK_P>(st, sp, grid, smem);
      case SK_M: return launch_sweep_t<T, GK_A, SK_M>(st, sp, grid, smem);
      case SK_F: return launch_sweep_t<T, GK_A, SK_F>(st, sp, grid, smem);
      case SK_R: return launch_sweep_t<T, GK_A, SK_R>(st, sp, grid, smem);
      case SK_L: return launch_sweep_t<T, GK_A, SK_L>(st, sp, grid, smem);
      case SK_Q: return launch_sweep_t<T, GK_A, SK_Q>(st, sp, grid, smem);
      case SK_N: return launch_sweep_t<T, GK_A, SK_N>(st, sp, grid, smem);
    }
  } else if (gk == GK_H) {
    switch (sk) {
      case SK_P: return launch_sweep_t<T, GK_H, SK_P>(st, sp, grid, smem);
      case SK_M: return launch_sweep_t<T, GK_H, SK_M>(st, sp, grid, smem);
      case SK_F: return launch_sweep_t<T, GK_H, SK_F>(st, sp, grid, smem);
    }
  } else if constexpr (sizeof(T) == 4) {
    switch (sk) {
      case SK_P: return launch_sweep_t<T, GK_H4, SK_P>(st, sp, grid, smem);
      case SK_M: return launch_sweep_t<T, GK_H4, SK_M>(st, sp, grid, smem);
      case SK_F: return launch_sweep_t<T, GK_H4, SK_F>(st, sp, grid, smem);
    }
  }
  return fail(LRQ_ERUNTIME, "internal: no sweep kernel for this (group, kind)");
}

int sm_count(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0) v = 148;
  return v;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

std::string gib(double bytes) {
  char b[64];
  snprintf(b, sizeof b, "%.1f", bytes / (double)(1ull << 30));
  return b;
}

}  // namespace

// In-process shard group: the shards of one state vector driven by host
// threads of one process (run_circuit_sharded, sharded.py:202-385), on one or
// several devices.  It replaces NCCL for these shards: the host barrier
// orders the streams, and the remap is a device-side swap of the shards'
// blocks (peer access across devices).  Any failure inside a collective
// call breaks the group for good (the reference's AbortedRunError).
struct lrq_group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int count = 0;
  unsigned long long gen = 0;
  bool broken = false;
  std::string why;
  std::vector<lrq_state*> members;
  std::vector<double> gather;               // 4 * world finalize scalars
  std::vector<const uint64_t*> shot_bufs;  // per-rank host sample buffers
  // fused remap decision, taken once every member exists (group_prepare):
  // second state buffers for all members, or none
  bool decided = false, fused_ok = false;
};

struct lrq_state {
  int n = 0;
  int pbytes = 0;
  int device = 0;
  int K = 13;  // tile amp bits
  cudaStream_t stream = nullptr;
  void* amps = nullptr;
  size_t state_bytes = 0;
  long long num_tiles = 1;
  double* red = nullptr;     // 4 arrays of num_tiles (p, pE, minE, arg bits)
  double* prefix = nullptr;  // num_tiles + 1
  double* out = nullptr;     // kOutScalars finalize scalars
  double* fin = nullptr;     // 5 * kFinBlocks finalize scratch
  double* dW = nullptr;      // n*n cost matrix
  double* dzero = nullptr;   // n zeros (no global qubits on a single device)
  double* dJ = nullptr;      // p*n*n phase matrices
  double* dmix = nullptr;    // p*2 (cos h, -sin h)
  int jcap = 0;
  double* du = nullptr;
  unsigned long long* didx = nullptr;
  long long shot_cap = 0;
  bool have_cost = false, reduced = false, ran = false;
  double wtot = 0.0;
  bool timing = false;
  std::vector<cudaEvent_t> evs;
  std::vector<char> kinds;
  std::vector<double> last_ms;
  // distributed (world > 1): n above is the local qubit count n_total - g
  int world = 1, rank = 0, g = 0, n_total = 0;
  ncclComm_t comm = nullptr;
  lrq_group* group = nullptr;      // in-process transport (lrq_create_shard)
  // fused remap: two state buffers per rank (amps == bufs[cur]); the sweep
  // before a remap writes the next buffer of every rank through peer pointers
  void* bufs[2] = {nullptr, nullptr};  // bufs[0] = the primary buffer (always), bufs[1] = fused-remap spare
  int cur = 0;
  void* peer[2][8] = {};  // peers' buffers (NCCL ranks: IPC-mapped; world <= 8)
  bool fused = false;     // fused remap: both buffers of every rank mapped and tested
  bool peer_ok = false;   // pipelined remap over peer memory: primary buffers mapped and tested
  std::vector<void*> ipc_open;  // peer buffers mapped with cudaIpcOpenMemHandle
  float* dflag = nullptr;       // 2 floats: NCCL stream barrier / pair token (send, recv)
  float* probe = nullptr;       // IPC self-test target (world floats)
  unsigned char* stage = nullptr;  // NCCL remap staging, chunk bytes
  size_t chunk = 0;
  cudaStream_t cstream = nullptr;  // remap stream (pipelined exchange, overlapped with the sweep)
  std::vector<cudaEvent_t> pev;    // world + 1 events: block j of the remap sweep done / remap done
  bool broken = false;             // a collective failed: the communicator was aborted
  std::vector<double> cost_edges;  // global cost edges (lexicographic)
  double* dWx = nullptr;           // cost field from the rank's qubits (n_loc), identity layout
  double wcst = 0.0;
  // the cost in the swapped layout (global <-> top local qubits): the final
  // pass of an odd-p run, and reductions before the layout is restored
  double* dW1 = nullptr;
  double* dWx1 = nullptr;
  double wcst1 = 0.0;
  int layout = 0;  // permutation state of the stored amplitudes (distributed states)
  double* dgather = nullptr;       // 4 * world doubles (all-gathered reductions)
  // optional per-layer Z fields / constant phases (lrq_run_fields)
  std::vector<double> field_h, cst_h;
  // optional per-qubit mixer signs relative to the layer angle (lrq_run_ex)
  std::vector<signed char> msign_h;
  signed char* dmsign = nullptr;
  size_t msign_cap = 0;
  double* dF = nullptr;
  int fcap = 0;
  std::vector<double> rank_sum_p;  // per-rank probability mass of the last run
  double remap_ms = 0.0;
  // p-weighted energy histogram of the reducing passes (lrq_set_histogram)
  unsigned long long* dhist = nullptr;
  int hist_bins = 0;
  double hist_lo = 0.0, hist_hi = 0.0;
  bool hist_summed = false;  // NCCL ranks: dhist already holds the sum over ranks
  bool hist_valid = false;   // a reducing pass has filled dhist since lrq_set_histogram
  bool search = true;        // reducing passes search min E / argmin / max E (lrq_set_search)
};

namespace {

void free_state(lrq_state* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  for (void* p : s->ipc_open) cudaIpcCloseMemHandle(p);
  if (s->bufs[0]) {
    cudaFree(s->bufs[0]);
    cudaFree(s->bufs[1]);
  } else {
    cudaFree(s->amps);
  }
  cudaFree(s->dflag);
  cudaFree(s->probe);
  for (cudaEvent_t e : s->pev) cudaEventDestroy(e);
  if (s->cstream) cudaStreamDestroy(s->cstream);
  cudaFree(s->red);
  cudaFree(s->prefix);
  cudaFree(s->out);
  cudaFree(s->fin);
  cudaFree(s->dW);
  cudaFree(s->dzero);
  cudaFree(s->dJ);
  cudaFree(s->dmix);
  cudaFree(s->du);
  cudaFree(s->didx);
  cudaFree(s->stage);
  cudaFree(s->dWx);
  cudaFree(s->dW1);
  cudaFree(s->dWx1);
  cudaFree(s->dF);
  cudaFree(s->dmsign);
  cudaFree(s->dgather);
  cudaFree(s->dhist);
  if (s->comm && nccl().ok) nccl().CommDestroy(s->comm);
  if (s->group) {
    std::lock_guard<std::mutex> lk(s->group->mu);
    if (s->rank < (int)s->group->members.size() && s->group->members[s->rank] == s)
      s->group->members[s->rank] = nullptr;
  }
  for (cudaEvent_t e : s->evs) cudaEventDestroy(e);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

// sequential v_n: n products by fl(1/sqrt 2) in the state precision
// (reference H kernel applied to |0..0>, engine.py:128-134)
template <typename T>
double init_amplitude(int n) {
  const T r = (T)(1.0 / sqrt(2.0));
  T v = (T)1.0;
  for (int i = 0; i < n; ++i) v = v * r;
  return (double)v;
}

void sym_matrix(int n, const double* e, double* M) {
  memset(M, 0, sizeof(double) * n * n);
  int k = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j, ++k) M[i * n + j] = M[j * n + i] = e[k];
}

// RX(theta) = cos(h) I - i sin(h) X = c I + i s X, h = theta/2 (engine.py:137-144).
// |s| <= |c|:  c (I + i t X) with t = s/c                      (flip = 0)
// |s| >  |c|:  (i s) X (I + i t X) with t = -c/s               (flip = 1)
// A layer applies the mixer to every qubit, so a flipped layer contributes
// X^(x)n, which commutes with every cost phase (E(~z) = E(z)) and mixer: it is
// deferred to one global index reversal at the end of the run.
struct MixerForm {
  double t;
  int flip;
  double qre, qim;  // per-qubit scalar factor
};
MixerForm mixer_form(double h) {
  const double c = cos(h), s = -sin(h);
  MixerForm f;
  if (fabs(s) <= fabs(c)) {
    f.t = s / c;
    f.flip = 0;
    f.qre = c;
    f.qim = 0.0;
  } else {
    f.t = -c / s;
    f.flip = 1;
    f.qre = 0.0;
    f.qim = s;
  }
  return f;
}

// tangents with per-qubit signs (lrq_run_ex): slot a of round r mixes qubit
// sweep_qubit(...); returns the number of mixed qubits whose sign is -1
int fill_tangents_signed(SweepParams& sp, int w, const PlanGroup& g, const PlanSweep& sw, int pair,
                         const unsigned* masks, double t, const signed char* sign) {
  int neg = 0;
  for (int r = 0; r < sw.nrounds; ++r)
    for (int a = 0; a < 5; ++a) {
      double v = 0.0;
      if ((masks[r] >> a) & 1u) {
        const int q = sweep_qubit(g, sw, pair, r, a);
        v = sign[q] < 0 ? -t : t;
        neg += sign[q] < 0;
      }
      sp.tf[w][r][a] = (float)v;
      sp.td[w][r][a] = v;
    }
  return neg;
}

void fill_tangents(SweepParams& sp, int w, const unsigned* masks, int nrounds, double t) {
  for (int r = 0; r < nrounds; ++r)
    for (int a = 0; a < 5; ++a) {
      const double v = ((masks[r] >> a) & 1u) ? t : 0.0;
      sp.tf[w][r][a] = (float)v;
      sp.td[w][r][a] = v;
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Tensor map over the runs of an H-group tile, in 8-byte elements:
//   d0 = run (2^MA amps), d1 = block bits below q0, d2/d3 = run index bits
//   (strides 2^q0 amps), d4 = block bits above the run index.
// Tensor map whose box is one whole 64 KB tile in natural tile order, with
// the 128B swizzle the TMA sweep kernel reads (8-byte elements):
//   A (contiguous):  {16, 256, 2T} box {16, 256, 2}
//   H complex64:     {2^MA, 32 runs, 2^(q0-MA) block, 2^(nrb-5) runs, rest} box {2^MA, 32, 1, 2^(nrb-5), 1}
//   H complex128:    {16, 2, 2^(q0-4) block, 256 runs, rest}            box {16, 2, 1, 256, 1}
// Coordinates of tile tid: A (0, 0, 2 tid); H (0, 0, tid_low, 0, tid_high).
bool make_tile_tmap(CUtensorMap* tm, void* amps, int gk, int n, int pbytes, int MA, int KA, int q0,
                    long long num_tiles) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return false;
  const cuuint64_t B = (cuuint64_t)pbytes;
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  if (gk == GK_A) {
    cuuint64_t dims[3] = {16, 256, 2ull * (cuuint64_t)num_tiles};
    cuuint64_t strides[2] = {128, 32768};
    cuuint32_t box[3] = {16, 256, 2};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const int nrb = KA - MA;
  if (pbytes == 8 && MA >= 5) {
    // cluster groups with runs longer than the 128 B swizzle span: each run is
    // 2^(MA-4) rows of 16 elements (like the complex128 H tile), natural order
    cuuint64_t dims[5] = {16, 1ull << (MA - 4), 1ull << (q0 - MA), 1ull << nrb, 1ull << (n - q0 - nrb)};
    cuuint64_t strides[4] = {128, (1ull << MA) * B, (1ull << q0) * B, (1ull << (q0 + nrb)) * B};
    cuuint32_t box[5] = {16, (cuuint32_t)(1u << (MA - 4)), 1, (cuuint32_t)(1u << nrb), 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  if (pbytes == 8) {
    // 64 B runs (MA = 3) use the 64B swizzle: a swizzled box row is padded
    // to the swizzle width, so 64 B rows under the 128B mode would not fit
    cuuint64_t dims[5] = {1ull << MA, 32, 1ull << (q0 - MA), 1ull << (nrb - 5), 1ull << (n - q0 - nrb)};
    cuuint64_t strides[4] = {(1ull << q0) * B, (1ull << MA) * B, (1ull << (q0 + 5)) * B, (1ull << (q0 + nrb)) * B};
    cuuint32_t box[5] = {(cuuint32_t)(1u << MA), 32, 1, (cuuint32_t)(1u << (nrb - 5)), 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              MA == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  cuuint64_t dims[5] = {16, 2, 1ull << (q0 - MA), 1ull << nrb, 1ull << (n - q0 - nrb)};
  cuuint64_t strides[4] = {128, (1ull << MA) * B, (1ull << q0) * B, (1ull << (q0 + nrb)) * B};
  cuuint32_t box[5] = {16, 2, 1, (cuuint32_t)(1u << nrb), 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, amps, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void cpow_mul(double& re, double& im, double qre, double qim, int k) {
  for (int i = 0; i < k; ++i) {
    const double r = re * qre - im * qim, m = re * qim + im * qre;
    re = r;
    im = m;
  }
}

template <typename T, int GK, int SK, int TEAMS>
int launch_tma_t(cudaStream_t st, const SweepParams& sp, int grid, size_t smem) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(sweep_tma_kernel<T, GK, SK, TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
  });
  CUDA_TRY(err);
  sweep_tma_kernel<T, GK, SK, TEAMS><<<grid, TEAMS * kThreads, smem, st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  return LRQ_OK;
}

template <typename T, int GK, int TEAMS>
int launch_tma_kind(cudaStream_t st, int sk, const SweepParams& sp, int grid, size_t smem) {
  switch (sk) {
    case SK_M: return launch_tma_t<T, GK, SK_M, TEAMS>(st, sp, grid, smem);
    case SK_F: return launch_tma_t<T, GK, SK_F, TEAMS>(st, sp, grid, smem);
  }
  if constexpr (GK == GK_A) {
    switch (sk) {
      case SK_R: return launch_tma_t<T, GK, SK_R, TEAMS>(st, sp, grid, smem);
      case SK_L: return launch_tma_t<T, GK, SK_L, TEAMS>(st, sp, grid, smem);
      case SK_Q: return launch_tma_t<T, GK, SK_Q, TEAMS>(st, sp, grid, smem);
    }
  }
  return fail(LRQ_ERUNTIME, "internal: no TMA sweep kernel for this (group, kind)");
}

template <typename T, int TEAMS>
int launch_tma_any(cudaStream_t st, int gk, int sk, const SweepParams& sp, int grid, size_t smem) {
  if (gk == GK_A) return launch_tma_kind<T, GK_A, TEAMS>(st, sk, sp, grid, smem);
  if (gk == GK_H) return launch_tma_kind<T, GK_H, TEAMS>(st, sk, sp, grid, smem);
  if constexpr (sizeof(T) == 4) return launch_tma_kind<T, GK_H4, TEAMS>(st, sk, sp, grid, smem);
  return fail(LRQ_ERUNTIME, "internal: no complex128 H4 group");
}

// Which sweeps take the TMA-fed pipeline: $LRQ_SWEEP_PATH = "reg" (none),
// "tma" (all that load), or a list of "<precision><group><kind>" tokens; the
// default keeps each sweep on the path measured faster on B200
// (profiles/r01_*): complex64 M and F on high groups.
bool use_tma_path(int pbytes, int gk, int sk) {
  if (sk == SK_P || sk == SK_N) return false;
  const char* v = getenv("LRQ_SWEEP_PATH");
  if (v && strcmp(v, "reg") == 0) return false;
  if (v && strcmp(v, "tma") == 0) return true;
  const char* g = gk == GK_A ? "A" : (gk == GK_H4 ? "H4" : "H");
  char tok[16];
  snprintf(tok, sizeof tok, "%s%s%c", pbytes == 8 ? "c64" : "c128", g, "PMFRLQN"[sk]);
  if (v && *v) return strstr(v, tok) != nullptr;
  return pbytes == 8 && gk != GK_A && (sk == SK_M || sk == SK_F);
}

template <typename T, int GK, int SK, int TEAMS>
int launch_wd_t(cudaStream_t st, const SweepParams& sp, int grid, size_t smem) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(sweep_wd_kernel<T, GK, SK, TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
  });
  CUDA_TRY(err);
  sweep_wd_kernel<T, GK, SK, TEAMS><<<grid, TEAMS * kWdWarps * 32, smem, st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  return LRQ_OK;
}

// P (no load, light on registers) runs three tiles in flight, each team on
// its own stage; M and F keep two so their threads get 255 registers
template <typename T, int GK>
int launch_wd_kind(cudaStream_t st, int sk, const SweepParams& sp, int grid, size_t smem) {
  if (sk == SK_F) return launch_wd_t<T, GK, SK_F, 2>(st, sp, grid, smem);
  if (sk == SK_P) return launch_wd_t<T, GK, SK_P, 3>(st, sp, grid, smem);
  return launch_wd_t<T, GK, SK_M, 2>(st, sp, grid, smem);
}

// warp-decoupled high-group sweep (plan prog 1): TMA ring of 3 stages, 2
// tiles in flight, one CTA per SM
int launch_wd(lrq_state* s, int gk, int sk, const SweepParams& sp_in) {
  SweepParams sp = sp_in;
  const int K = tile_amp_bits(s->pbytes);
  const int ma = group_ma(gk, pair_of(s->pbytes));
  if (!make_tile_tmap(&sp.tmap, sp.amps, gk, sp.n, s->pbytes, ma, K, sp.q0, sp.num_tiles))
    return fail(LRQ_ERUNTIME, "cuTensorMapEncodeTiled failed for the sweep tile map");
  sp.has_tmap = 1;
  sp.nstages = 3;
  // measured: +1-2 % on H groups, -35 % on H4 (its 512-row tensor prefetch
  // competes with the ring's own loads and stores)
  sp.wd_prefetch = env_int("LRQ_WD_PREFETCH", gk == GK_H ? 1 : 0);
  const size_t smem = wd_smem_bytes(sp.n, 3, sk == SK_F || sk == SK_P);
  if (smem > 227 * 1024) return fail(LRQ_ERUNTIME, "internal: warp-decoupled sweep needs too much shared memory");
  const int sms = sm_count(s->device);
  const int g = (int)(sp.num_tiles < sms ? sp.num_tiles : sms);
  if (s->pbytes == 16) {
    if (gk != GK_H) return fail(LRQ_ERUNTIME, "internal: complex128 warp-decoupled sweeps need an H group");
    return launch_wd_kind<double, GK_H>(s->stream, sk, sp, g, smem);
  }
  if (gk == GK_H) return launch_wd_kind<float, GK_H>(s->stream, sk, sp, g, smem);
  return launch_wd_kind<float, GK_H4>(s->stream, sk, sp, g, smem);
}

template <int GK, int SK, int TEAMS>
int launch_wdc_t(cudaStream_t st, const SweepParams& sp, int grid, size_t smem) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(sweep_wdc_kernel<GK, SK, TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
  });
  CUDA_TRY(err);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(TEAMS * kWdWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;  // the CTA pair sharing one 128 KB tile
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, sweep_wdc_kernel<GK, SK, TEAMS>, sp));
  return LRQ_OK;
}

template <int GK>
int launch_wdc_kind(cudaStream_t st, int sk, const SweepParams& sp, int grid, size_t smem) {
  if (sk == SK_F) return launch_wdc_t<GK, SK_F, 2>(st, sp, grid, smem);
  if (sk == SK_P) return launch_wdc_t<GK, SK_P, 2>(st, sp, grid, smem);  // 2 teams: 255 registers, no spills
  return launch_wdc_t<GK, SK_M, 2>(st, sp, grid, smem);
}

// cluster-pair sweep of a complex64 C group (plan prog 2): 148 CTAs = 74
// pairs, each pair one 128 KB tile at a time, three 64 KB stages per CTA
int launch_wdc(lrq_state* s, int gk, int sk, const SweepParams& sp_in) {
  SweepParams sp = sp_in;
  const int K = tile_amp_bits(s->pbytes);
  const int ma = group_ma(gk, pair_of(s->pbytes));
  if (s->pbytes != 8) return fail(LRQ_ERUNTIME, "internal: cluster groups are complex64");
  if (!make_tile_tmap(&sp.tmap, sp.amps, gk, sp.n, s->pbytes, ma, K, sp.q0, sp.num_tiles))
    return fail(LRQ_ERUNTIME, "cuTensorMapEncodeTiled failed for the cluster sweep tile map");
  sp.has_tmap = 1;
  sp.nstages = 3;
  const size_t smem = wdc_smem_bytes(sp.n, 3, sk == SK_F || sk == SK_P);
  if (smem > 227 * 1024) return fail(LRQ_ERUNTIME, "internal: cluster sweep needs too much shared memory");
  int g = sm_count(s->device) & ~1;
  const long long pairs = sp.num_tiles / 2;
  if (pairs < g / 2) g = (int)(2 * pairs);
  if (g < 2) return fail(LRQ_ERUNTIME, "internal: cluster sweep needs at least one tile pair");
  switch (gk) {
    case GK_C10: return launch_wdc_kind<GK_C10>(s->stream, sk, sp, g, smem);
    case GK_C9: return launch_wdc_kind<GK_C9>(s->stream, sk, sp, g, smem);
    case GK_C8: return launch_wdc_kind<GK_C8>(s->stream, sk, sp, g, smem);
  }
  return fail(LRQ_ERUNTIME, "internal: not a cluster group");
}

int launch_sweep(lrq_state* s, int gk, int sk, const SweepParams& sp_in, int grid) {
  const bool amps = sk != SK_N;
  const bool usesJ = sk == SK_P || sk == SK_F || sk == SK_L;
  const bool usesW = sk == SK_R || sk == SK_Q || sk == SK_N || (sk == SK_L && sp_in.reduce);
  if (!sp_in.hist && use_tma_path(s->pbytes, gk, sk)) {
    // TMA-fed pipeline: one CTA per SM, a ring of 64 KB stages, 1 or 2 teams
    SweepParams sp = sp_in;
    const int K = tile_amp_bits(s->pbytes);
    const int ma = group_ma(gk, pair_of(s->pbytes));
    if (!make_tile_tmap(&sp.tmap, sp.amps, gk, sp.n, s->pbytes, ma, K, sp.q0, sp.num_tiles))
      return fail(LRQ_ERUNTIME, "cuTensorMapEncodeTiled failed for the sweep tile map");
    sp.has_tmap = 1;
    const size_t cap = 227 * 1024;
    // F sweeps (two mixers + phase) overlap better with two independent teams;
    // the lighter M sweeps stream best with one team and 255 registers
    int teams = env_int("LRQ_TMA_TEAMS", sk == SK_F ? 2 : 1);
    teams = teams == 1 ? 1 : 2;
    if (teams == 2 && tma_smem_bytes(sp.n, 3, 2, usesJ, usesW) > cap) teams = 1;
    sp.nstages = tma_smem_bytes(sp.n, 3, teams, usesJ, usesW) <= cap ? 3 : 2;
    const size_t smem = tma_smem_bytes(sp.n, sp.nstages, teams, usesJ, usesW);
    const int sms = sm_count(s->device);
    const int g = (int)(sp.num_tiles < sms ? sp.num_tiles : sms);
    if (s->pbytes == 8)
      return teams == 2 ? launch_tma_any<float, 2>(s->stream, gk, sk, sp, g, smem)
                        : launch_tma_any<float, 1>(s->stream, gk, sk, sp, g, smem);
    return teams == 2 ? launch_tma_any<double, 2>(s->stream, gk, sk, sp, g, smem)
                      : launch_tma_any<double, 1>(s->stream, gk, sk, sp, g, smem);
  }
  const size_t smem = sweep_smem_bytes(sp_in.n, amps, usesJ, usesW, sp_in.hist ? sp_in.hist_bins : 0);
  if (s->pbytes == 8) return launch_sweep_kind<float>(s->stream, gk, sk, sp_in, grid, smem);
  return launch_sweep_kind<double>(s->stream, gk, sk, sp_in, grid, smem);
}

// deterministic combine of the per-tile partials + CDF prefix (lrq_aux.cuh);
// bs: kFinScratch doubles of scratch (multi-CTA path for large T)
int launch_finalize(cudaStream_t st, long long T, double* red, double* prefix, double* out, double* bs) {
  double* rp = red;
  double* rpe = red + T;
  double* rmin = red + 2 * T;
  unsigned long long* rarg = reinterpret_cast<unsigned long long*>(red + 3 * T);
  const double* rmax = red + 4 * T;
  if (T < 8192 || !bs) {
    finalize_kernel<<<1, 1024, 0, st>>>(T, rp, rpe, rmin, rarg, rmax, prefix, out);
    CUDA_TRY(cudaGetLastError());
    return LRQ_OK;
  }
  const long long per = (T + kFinBlocks - 1) / kFinBlocks;
  const int nb = (int)((T + per - 1) / per);
  finalize_blocks<<<nb, 256, 0, st>>>(T, per, rp, rpe, rmin, rarg, rmax, prefix, bs);
  CUDA_TRY(cudaGetLastError());
  finalize_combine<<<1, 32, 0, st>>>(nb, T, bs, prefix, out);
  CUDA_TRY(cudaGetLastError());
  finalize_offsets<<<nb, 256, 0, st>>>(T, per, bs, prefix);
  CUDA_TRY(cudaGetLastError());
  return LRQ_OK;
}

template <typename T>
int launch_small(const SmallParams& sp, size_t smem, cudaStream_t st, int grid = 1) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(small_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  });
  CUDA_TRY(err);
  small_kernel<T><<<grid, 256, smem, st>>>(sp);
  CUDA_TRY(cudaGetLastError());
  return LRQ_OK;
}

int launch_small_any(int pbytes, const SmallParams& sp, cudaStream_t st) {
  const size_t smem = (size_t)pbytes * (1u << sp.n) + 8 * 5 * 8;
  return pbytes == 8 ? launch_small<float>(sp, smem, st) : launch_small<double>(sp, smem, st);
}

void record(lrq_state* s, size_t idx, char kind) {
  if (!s->timing) return;
  while (s->evs.size() <= idx) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    s->evs.push_back(e);
  }
  cudaEventRecord(s->evs[idx], s->stream);
  if (kind) s->kinds.push_back(kind);
}

// the energy histogram of a reducing pass (lrq_set_histogram): zeroed on
// the engine stream before the pass, filled by the pass's integer atomics
template <typename PR>
void set_hist(lrq_state* s, PR& sp) {
  sp.search = s->search ? 1 : 0;
  if (!s->dhist) return;
  s->hist_valid = true;  // filled by the pass being set up
  sp.hist = s->dhist;
  sp.hist_bins = s->hist_bins;
  sp.hist_lo = s->hist_lo;
  sp.hist_scale = s->hist_bins / (s->hist_hi - s->hist_lo);
}
int zero_hist(lrq_state* s) {
  s->hist_summed = false;
  if (s->dhist) CUDA_TRY(cudaMemsetAsync(s->dhist, 0, sizeof(unsigned long long) * s->hist_bins, s->stream));
  return LRQ_OK;
}

#define NCCL_TRY(expr)                                                                           \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return fail(LRQ_ERUNTIME, std::string("NCCL error in ") + #expr + ": " + nccl().GetErrorString(r_)); \
  } while (0)

// Host barrier of an in-process group (600 s limit, like the reference's
// receive timeout, sharded.py:38).
int group_barrier(lrq_group* G) {
  std::unique_lock<std::mutex> lk(G->mu);
  if (G->broken) return fail(LRQ_ERUNTIME, "aborted run: shard group: " + G->why);
  const unsigned long long my = G->gen;
  if (++G->count == G->world) {
    G->count = 0;
    ++G->gen;
    G->cv.notify_all();
    return LRQ_OK;
  }
  if (!G->cv.wait_for(lk, std::chrono::seconds(600), [&] { return G->gen != my || G->broken; })) {
    G->broken = true;
    G->why = "barrier timeout";
    G->cv.notify_all();
  }
  if (G->gen == my) return fail(LRQ_ERUNTIME, "aborted run: shard group: " + G->why);
  return LRQ_OK;
}

void group_abort(lrq_group* G, const std::string& why) {
  std::lock_guard<std::mutex> lk(G->mu);
  if (!G->broken) G->why = why;
  G->broken = true;
  G->cv.notify_all();
}

// a[i] <-> b[i] over `units` 16-byte units; four independent pairs per
// thread and iteration keep enough NVLink reads in flight for a peer buffer
__global__ void __launch_bounds__(256) swap_kernel(uint4* __restrict__ a, uint4* __restrict__ b, long long units) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < units; i += 4 * stride) {
    const uint4 x0 = a[i], x1 = a[i + stride], x2 = a[i + 2 * stride], x3 = a[i + 3 * stride];
    const uint4 y0 = b[i], y1 = b[i + stride], y2 = b[i + 2 * stride], y3 = b[i + 3 * stride];
    a[i] = y0;
    a[i + stride] = y1;
    a[i + 2 * stride] = y2;
    a[i + 3 * stride] = y3;
    b[i] = x0;
    b[i + stride] = x1;
    b[i + 2 * stride] = x2;
    b[i + 3 * stride] = x3;
  }
  for (; i < units; i += stride) {
    const uint4 x = a[i], y = b[i];
    a[i] = y;
    b[i] = x;
  }
}

int enable_peer(int dev, int peer) {
  if (dev == peer) return LRQ_OK;
  int ok = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&ok, dev, peer));
  if (!ok) return fail(LRQ_ERUNTIME, "shard group spans devices without peer access");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);  // on the current device (dev)
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return LRQ_OK;
  }
  CUDA_TRY(e);
  return LRQ_OK;
}

// ---------------------------------------------------------------------------
// Failure handling of NCCL ranks (reference: a failed shard worker aborts the
// whole run with AbortedRunError, sharded.py:328-349).  Every wait on a
// stream that carries collectives polls the communicator's async error and a
// wall-clock limit ($LRQ_DIST_TIMEOUT_S, default 600 s like the reference's
// receive timeout, sharded.py:38); on either the communicator is aborted
// (ncclCommAbort, which also unblocks the NCCL kernels of this rank) and the
// state refuses further collectives.
int abort_comm(lrq_state* s, const std::string& why) {
  if (s->comm && nccl().ok) nccl().CommAbort(s->comm);
  s->comm = nullptr;
  s->broken = true;
  return fail(LRQ_ERUNTIME, "aborted run: " + why);
}

int dist_wait(lrq_state* s, cudaStream_t st) {
  if (!s->comm) {
    if (s->broken) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
    CUDA_TRY(cudaStreamSynchronize(st));
    return LRQ_OK;
  }
  const double limit = (double)env_int("LRQ_DIST_TIMEOUT_S", 600);
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned it = 0;; ++it) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return LRQ_OK;
    if (e != cudaErrorNotReady) return abort_comm(s, std::string("CUDA error: ") + cudaGetErrorString(e));
    ncclResult_t ae = ncclSuccess;
    if (nccl().CommGetAsyncError(s->comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress)
      return abort_comm(s, std::string("NCCL error on another rank or link: ") + nccl().GetErrorString(ae));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > limit) return abort_comm(s, "no progress from the other ranks for " + std::to_string((int)limit) + " s");
    if (it > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

#define NCCL_TRY_S(s, expr)                                                                          \
  do {                                                                                               \
    ncclResult_t r_ = (expr);                                                                        \
    if (r_ != ncclSuccess) return abort_comm((s), std::string("NCCL error in ") + #expr + ": " +    \
                                                      nccl().GetErrorString(r_));                     \
  } while (0)

int ensure_remap_stream(lrq_state* s) {
  if (!s->cstream) CUDA_TRY(cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking));
  while ((int)s->pev.size() < s->world + 1) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    s->pev.push_back(e);
  }
  return LRQ_OK;
}

// One pairwise step of a remap on rank `rank`: swap my block my_block with
// block their_block of `partner`; half = 0 / 1: the half of the pair's bytes
// this rank moves in a peer-memory swap (lower rank: first half).
struct RemapStep {
  int partner;
  int my_block, their_block;  // in blocks of the remap (-1: the whole state, the mirror exchange)
  int half;
};
// XOR schedule of the all-to-all block transpose (step k = 1..world-1:
// partner rank ^ k), or the single mirror step of the deferred global flip.
inline std::vector<RemapStep> remap_schedule(int world, int rank, int mirror) {
  std::vector<RemapStep> v;
  if (mirror >= 0) {
    v.push_back({mirror, -1, -1, rank < mirror ? 0 : 1});
    return v;
  }
  for (int k = 1; k < world; ++k) {
    const int p = rank ^ k;
    v.push_back({p, p, rank, rank < p ? 0 : 1});
  }
  return v;
}

// Remap transports.  A remap swaps the g global qubits with the top g local
// bits: local block b (top g local bits = b) of rank r trades places with
// block r of rank b — an all-to-all block transpose done in place as G-1
// pairwise swaps on the XOR schedule (step k: rank r <-> r ^ k; every rank has
// exactly one partner per step, and block r^k of r pairs with block r of r^k).
// `mirror` >= 0 instead swaps the whole local state with that one rank (the
// deferred global flip).  Transports, chosen at setup:
//   group  in-process shards: a swap kernel over the members' buffers (same
//          device or peer access); host barriers order the ranks;
//   peer   NCCL ranks whose primary buffers are IPC-mapped: a 1-float
//          send/recv token pairs the two ranks, then each swaps its half of
//          the two blocks in place over NVLink (no staging, no copy);
//   nccl   otherwise: chunked ncclSend/ncclRecv into one staging chunk, then
//          a device copy into the block.
// Each rank calls pair_exchange with mirrored offsets; the lower rank of the
// pair takes the first half of a peer-memory swap, the higher one the rest.
int pair_exchange(lrq_state* s, int p, size_t my_off, size_t their_off, size_t bytes, int which_half,
                  cudaStream_t st) {
  unsigned char* mine = reinterpret_cast<unsigned char*>(s->amps) + my_off;
  const int grid = 2 * sm_count(s->device);
  if (s->group || s->peer_ok) {
    unsigned char* theirs = nullptr;
    if (s->group) {
      lrq_state* o = s->group->members[p];
      if (!o) return fail(LRQ_ERUNTIME, "aborted run: shard group member missing");
      const int rc = enable_peer(s->device, o->device);
      if (rc) return rc;
      theirs = reinterpret_cast<unsigned char*>(o->amps) + their_off;
    } else {
      // pair token: the partner has reached this step (its blocks are final)
      NCCL_TRY_S(s, nccl().GroupStart());
      NCCL_TRY_S(s, nccl().Send(s->dflag, 1, ncclFloat, p, s->comm, st));
      NCCL_TRY_S(s, nccl().Recv(s->dflag + 1, 1, ncclFloat, p, s->comm, st));
      NCCL_TRY_S(s, nccl().GroupEnd());
      theirs = reinterpret_cast<unsigned char*>(s->peer[0][p]) + their_off;
    }
    const size_t half = (bytes / 2) & ~(size_t)15;
    const size_t off = which_half == 0 ? 0 : half, len = which_half == 0 ? half : bytes - half;
    swap_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<uint4*>(mine + off), reinterpret_cast<uint4*>(theirs + off),
                                      (long long)(len / 16));
    CUDA_TRY(cudaGetLastError());
    return LRQ_OK;
  }
  NcclApi& nc = nccl();
  for (size_t o = 0; o < bytes; o += s->chunk) {
    const size_t len = bytes - o < s->chunk ? bytes - o : s->chunk;
    NCCL_TRY_S(s, nc.GroupStart());
    NCCL_TRY_S(s, nc.Send(mine + o, len, ncclUint8, p, s->comm, st));
    NCCL_TRY_S(s, nc.Recv(s->stage, len, ncclUint8, p, s->comm, st));
    NCCL_TRY_S(s, nc.GroupEnd());
    CUDA_TRY(cudaMemcpyAsync(mine + o, s->stage, len, cudaMemcpyDeviceToDevice, st));
  }
  return LRQ_OK;
}

// The whole remap (or the mirror exchange).  pipelined: the blocks come from
// a sweep split by block on the engine stream, block r^k marked by event
// pev[k]; the swaps run on the remap stream as the blocks complete, and the
// engine stream waits for the last one.  Otherwise the sweep has finished on
// the engine stream and the swaps follow on it.
int remap_exchange(lrq_state* s, bool pipelined, int mirror) {
  const bool grp = s->group != nullptr;
  if (!grp && !s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
  int rc = ensure_remap_stream(s);
  if (rc) return rc;
  cudaStream_t st = pipelined ? s->cstream : s->stream;
  const size_t block = (size_t)s->pbytes << (s->n - s->g), whole = (size_t)s->pbytes << s->n;
  if (grp && !pipelined) {
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    if ((rc = group_barrier(s->group))) return rc;
  }
  const std::vector<RemapStep> steps = remap_schedule(s->world, s->rank, mirror);
  for (int k = 1; k <= (int)steps.size(); ++k) {
    const RemapStep& sp = steps[k - 1];
    const int p = sp.partner;
    if (pipelined) {
      if (grp) {
        CUDA_TRY(cudaEventSynchronize(s->pev[k]));
        if ((rc = group_barrier(s->group))) return rc;
      } else {
        CUDA_TRY(cudaStreamWaitEvent(st, s->pev[k], 0));
      }
    }
    if (sp.my_block < 0) rc = pair_exchange(s, p, 0, 0, whole, sp.half, st);
    else rc = pair_exchange(s, p, (size_t)sp.my_block * block, (size_t)sp.their_block * block, block, sp.half, st);
    if (rc) return rc;
  }
  if (grp) {
    CUDA_TRY(cudaStreamSynchronize(st));
    return group_barrier(s->group);  // every member's swaps into our blocks are done
  }
  // peer transport: the partners write into our blocks; the all-reduce on the
  // same stream completes only after every rank's swap kernels
  if (s->peer_ok) NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, st));
  if (pipelined) {
    CUDA_TRY(cudaEventRecord(s->pev[s->world], st));
    CUDA_TRY(cudaStreamWaitEvent(s->stream, s->pev[s->world], 0));
  }
  return LRQ_OK;
}

// the sampler's sum over ranks for an in-process group (host buffers)
int group_sum_shots(lrq_state* s, uint64_t* idx, int64_t shots) {
  lrq_group* G = s->group;
  {
    std::lock_guard<std::mutex> lk(G->mu);
    G->shot_bufs[s->rank] = idx;
  }
  int rc = group_barrier(G);
  if (rc) return rc;
  std::vector<uint64_t> sum((size_t)shots, 0);
  for (int r = 0; r < G->world; ++r)
    for (int64_t k = 0; k < shots; ++k) sum[k] += G->shot_bufs[r][k];
  rc = group_barrier(G);
  if (rc) return rc;
  memcpy(idx, sum.data(), sizeof(uint64_t) * shots);
  return LRQ_OK;
}

// Device memory a rank needs besides the state: tile reductions + CDF prefix,
// finalize scratch, cost matrices, NCCL staging.  Host-side accounting shared
// by create_rank_state and lrq_describe_memory.
size_t remap_chunk(size_t block) { return block < (256ull << 20) ? block : (256ull << 20); }
size_t rank_extra_bytes(int n_loc, int pbytes, int world, int p, bool staging) {
  const long long T = n_loc >= tile_amp_bits(pbytes) ? (1ll << (n_loc - tile_amp_bits(pbytes))) : 1;
  int g = 0;
  while ((1 << g) < world) ++g;
  size_t b = 8ull * (4 * T + T + 1) + 8ull * (4 + 5 * kFinBlocks);     // red, prefix, out, fin
  b += 8ull * n_loc * n_loc + 8ull * (n_loc + 1) + 8ull * n_loc;        // dW, dzero, dWx
  b += 8ull * ((size_t)n_loc * n_loc + n_loc) * 2 * (p > 0 ? p : 1);     // dJ (both permutation states)
  b += 8ull * 4 * world + 2 * 4 + 4ull * world;                          // dgather, dflag, probe
  if (staging) b += remap_chunk((size_t)pbytes << (n_loc - g));
  return b;
}

// In-process groups: decide once, with every member present, whether all
// members get the second (fused-remap) buffer: only if, on every device, the
// members' spare buffers fit with 2 GiB to spare.  Otherwise no member gets
// one and remaps take the pipelined swap.
void group_prepare(lrq_state* s) {
  lrq_group* G = s->group;
  std::lock_guard<std::mutex> lk(G->mu);
  if (G->decided) return;
  for (lrq_state* m : G->members)
    if (!m) return;  // not every shard exists yet: decide later
  G->decided = true;
  G->fused_ok = false;
  if (!env_int("LRQ_FUSED_REMAP", 1) || G->world > 8) return;
  std::vector<int> devs;
  for (lrq_state* m : G->members)
    if (std::find(devs.begin(), devs.end(), m->device) == devs.end()) devs.push_back(m->device);
  for (int d : devs) {
    size_t need = 2ull << 30;
    for (lrq_state* m : G->members)
      if (m->device == d) need += m->state_bytes;
    DeviceGuard dg(d);
    size_t freeb = 0, totalb = 0;
    if (cudaMemGetInfo(&freeb, &totalb) != cudaSuccess || freeb < need) {
      cudaGetLastError();
      return;
    }
  }
  bool ok = true;
  for (lrq_state* m : G->members) {
    DeviceGuard dg(m->device);
    void* alt = nullptr;
    if (cudaMalloc(&alt, m->state_bytes) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    m->bufs[1] = alt;
  }
  if (!ok)
    for (lrq_state* m : G->members) {
      DeviceGuard dg(m->device);
      cudaFree(m->bufs[1]);
      m->bufs[1] = nullptr;
    }
  G->fused_ok = ok;
}

// fused remap availability: both state buffers on every rank and the peers'
// buffers addressable (in-process groups: the members' pointers, with peer
// access across devices; NCCL ranks: mapped by lrq_fused_setup)
bool fused_ready(lrq_state* s) {
  if (!env_int("LRQ_FUSED_REMAP", 1)) return false;
  if (s->group) {
    group_prepare(s);
    lrq_group* G = s->group;
    if (!G->fused_ok) return false;
    for (int b = 0; b < s->world; ++b) {
      lrq_state* o = G->members[b];
      if (!o || !o->bufs[1] || o->cur != s->cur) return false;
      if (o->device != s->device) {
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, s->device, o->device) != cudaSuccess || !ok) return false;
        cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return false;
        cudaGetLastError();
      }
      s->peer[0][b] = o->bufs[0];
      s->peer[1][b] = o->bufs[1];
    }
    return true;
  }
  return s->fused && s->bufs[1];
}

// all ranks' fused-remap stores are complete before anyone reads its buffer
int fused_barrier(lrq_state* s) {
  if (s->group) {
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    return group_barrier(s->group);
  }
  // stream-ordered: the all-reduce completes only after every rank's sweep
  NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, s->stream));
  return LRQ_OK;
}

// A rank's view of the cost in permutation state `perm` and the local bit
// that must be 0 in the max-cut search (the top logical qubit n-1: rank bit
// g-1 in the identity layout, local bit n_loc-1 in the swapped one).
MatArg cost_view(const lrq_state* s, int perm) {
  MatArg W;
  W.M = perm ? s->dW1 : s->dW;
  W.ext = perm ? s->dWx1 : s->dWx;
  W.cst = perm ? s->wcst1 : s->wcst;
  return W;
}
int search_bit(const lrq_state* s, int perm) {
  if (perm) return s->n - 1;
  return ((s->rank >> (s->g - 1)) & 1) ? -2 : -1;
}
// global basis index of local index z on rank `rank` (n_loc local qubits),
// in permutation `perm` (1: the top g local bits hold the global qubits and
// the rank bits the qubits [n_loc-g, n_loc))
uint64_t global_index(int nl, int g, int rank, int perm, uint64_t z) {
  if (!perm) return ((uint64_t)rank << nl) | z;
  const uint64_t low = z & ((1ull << (nl - g)) - 1ull), top = z >> (nl - g);
  return low | ((uint64_t)rank << (nl - g)) | (top << nl);
}

// lrq_run for world > 1 (make_dist_plan): local sweeps in the permutation
// state each one records, remaps between layers, final read-only reduction.
int run_dist(lrq_state* s, int p, const double* phase, const double* mixer) {
  const int nl = s->n, nt = s->n_total, g = s->g, E = nt * (nt - 1) / 2;
  const size_t per = (size_t)nl * nl + nl;
  if (2 * p > s->jcap) {
    cudaFree(s->dJ);
    s->dJ = nullptr;
    CUDA_TRY(cudaMalloc(&s->dJ, sizeof(double) * per * 2 * p));
    s->jcap = 2 * p;
  }
  std::vector<double> J(per * 2 * p), cst(2 * p);
  for (int k = 0; k < p; ++k)
    for (int perm = 0; perm < 2; ++perm) {
      double* dst = J.data() + per * (2 * k + perm);
      dist_terms(nt, g, s->rank, perm, phase + (size_t)k * E, dst, dst + (size_t)nl * nl, &cst[2 * k + perm]);
    }
  CUDA_TRY(cudaMemcpyAsync(s->dJ, J.data(), sizeof(double) * J.size(), cudaMemcpyHostToDevice, s->stream));
  const double init = s->pbytes == 8 ? init_amplitude<float>(nt) : init_amplitude<double>(nt);
  s->reduced = false;
  s->ran = false;
  s->kinds.clear();
  size_t ev = 0;
  record(s, ev++, 0);
  double* rp = s->red;
  double* rpe = rp + s->num_tiles;
  double* rmin = rpe + s->num_tiles;
  unsigned long long* rarg = reinterpret_cast<unsigned long long*>(rmin + s->num_tiles);
  double* rmax = rmin + 2 * s->num_tiles;
  const Plan P = make_dist_plan(nl, g, pair_of(s->pbytes), p);
  const int grid_cap = 2 * sm_count(s->device);
  const int grid = (int)(s->num_tiles < grid_cap ? s->num_tiles : grid_cap);
  int flips = 0;
  for (int k = 0; k < p; ++k) flips += mixer_form(mixer[k]).flip;
  const bool fused = fused_ready(s);
  for (const PlanSweep& w : P.sweeps) {
    const PlanGroup& gr = P.groups[w.group];
    if (w.kind == SK_Q && (flips & 1)) {
      // deferred X^(x)n of the flipped layers: z -> ~z reverses the local index
      // and maps rank r to rank world-1-r
      const long long half = (1ll << nl) / 2;
      const unsigned blocks = (unsigned)((half + 255) / 256);
      if (s->pbytes == 8) reverse_kernel<float2><<<blocks, 256, 0, s->stream>>>(s->amps, nl);
      else reverse_kernel<double2><<<blocks, 256, 0, s->stream>>>(s->amps, nl);
      CUDA_TRY(cudaGetLastError());
      int rc = remap_exchange(s, false, s->world - 1 - s->rank);
      if (rc) return rc;
      record(s, ev++, 'X');
    }
    SweepParams sp;
    memset(&sp, 0, sizeof sp);
    sp.amps = s->amps;
    sp.n = nl;
    sp.q0 = gr.q0;
    sp.num_tiles = s->num_tiles;
    sp.reduce = w.reduce ? 1 : 0;
    double sre = 1.0, sim = 0.0;
    if (w.beta1 >= 0) {
      const MixerForm f = mixer_form(mixer[w.beta1]);
      fill_tangents(sp, 0, w.mask1, w.nrounds, f.t);
      cpow_mul(sre, sim, f.qre, f.qim, w.ntarget1);
    }
    if (w.beta2 >= 0) {
      const MixerForm f = mixer_form(mixer[w.beta2]);
      fill_tangents(sp, 1, w.mask2, w.nrounds, f.t);
      cpow_mul(sre, sim, f.qre, f.qim, w.ntarget2);
    }
    sp.scale_re = sre;
    sp.scale_im = sim;
    sp.init_re = init;
    const double* jm = w.phase >= 0 ? s->dJ + per * (2 * w.phase + w.perm) : s->dW;
    sp.J.M = jm;
    sp.J.ext = w.phase >= 0 ? jm + (size_t)nl * nl : s->dzero;
    sp.J.cst = w.phase >= 0 ? cst[2 * w.phase + w.perm] : 0.0;
    sp.W = cost_view(s, w.perm);  // the final pass runs in the permutation the layers left
    sp.min_bit = search_bit(s, w.perm);
    sp.red_p = rp;
    sp.red_pE = rpe;
    sp.red_minE = rmin;
    sp.red_arg = rarg;
    sp.red_maxE = rmax;
    if (w.reduce) {
      if (const int rh = zero_hist(s)) return rh;
      set_hist(s, sp);
    }
    // (a tile must lie inside one destination block: n_loc - g >= tile bits)
    const bool fuse = w.remap_after && fused && gr.kind == GK_A && w.kind == SK_M && nl - g >= P.KA;
    if (fuse) {
      // the sweep stores block b of its output into rank b's next buffer at
      // this rank's block: the remap rides on the sweep's own stores
      const int next = 1 - s->cur;
      const size_t blockBytes = (size_t)s->pbytes << (nl - g);
      int tb = 0;
      while ((1ll << tb) < s->num_tiles) ++tb;
      sp.remap = 1;
      sp.rbits = tb - g;
      for (int b = 0; b < s->world; ++b) sp.rdst[b] = (char*)s->peer[next][b] + (size_t)s->rank * blockBytes;
    }
    const char kname[2] = {"PMFRLQN"[w.kind], 0};
    NvtxRange nv_sweep("sweep ", kname);
    // pipelined remap: the group-A sweep runs block by block in XOR order
    // (block rank ^ j at step j) and each finished block is swapped with its
    // owner while the next block is swept (remap_exchange on the remap stream)
    const bool pipe = !fuse && w.remap_after && gr.kind == GK_A && w.kind == SK_M && nl - g >= P.KA &&
                      env_int("LRQ_PIPELINED_REMAP", 1);
    int rc = LRQ_OK;
    if (pipe) {
      if ((rc = ensure_remap_stream(s))) return rc;
      const long long TB = s->num_tiles >> g;
      const size_t blockBytes = (size_t)s->pbytes << (nl - g);
      for (int j = 0; j < s->world && !rc; ++j) {
        SweepParams sb = sp;
        sb.amps = reinterpret_cast<char*>(s->amps) + (size_t)(s->rank ^ j) * blockBytes;
        sb.num_tiles = TB;
        rc = launch_sweep(s, gr.kind, w.kind, sb, (int)(TB < grid ? TB : grid));
        if (!rc && cudaEventRecord(s->pev[j], s->stream) != cudaSuccess)
          rc = fail(LRQ_ERUNTIME, "cudaEventRecord failed");
      }
      if (rc) return rc;
    } else {
      rc = w.prog == 1 ? launch_wd(s, gr.kind, w.kind, sp)
           : fuse      ? (s->pbytes == 8 ? launch_sweep_kind<float>(s->stream, gr.kind, w.kind, sp, grid,
                                                                     sweep_smem_bytes(nl, true, false, false))
                                         : launch_sweep_kind<double>(s->stream, gr.kind, w.kind, sp, grid,
                                                                      sweep_smem_bytes(nl, true, false, false)))
                       : launch_sweep(s, gr.kind, w.kind, sp, grid);
    }
    if (rc) return rc;
    record(s, ev++, "PMFRLQN"[w.kind]);
    if (fuse) {
      rc = fused_barrier(s);  // every rank's stores into our next buffer are done
      if (rc) return rc;
      s->cur = 1 - s->cur;
      s->amps = s->bufs[s->cur];
      record(s, ev++, 'Y');
    } else if (pipe) {
      NvtxRange nv_remap("remap pipelined");
      rc = remap_exchange(s, true, -1);
      if (rc) return rc;
      record(s, ev++, 'W');
    } else if (w.remap_after) {
      NvtxRange nv_remap("remap serial");
      rc = remap_exchange(s, false, -1);
      if (rc) return rc;
      record(s, ev++, 'T');
    }
  }
  {
    const int rc = launch_finalize(s->stream, s->num_tiles, s->red, s->prefix, s->out, s->fin);
    if (rc) return rc;
  }
  record(s, ev++, 'Z');
  {
    const int rc = dist_wait(s, s->stream);
    if (rc) return rc;
  }
  if (s->timing) {
    s->last_ms.clear();
    for (size_t i = 1; i < ev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, s->evs[i - 1], s->evs[i]);
      s->last_ms.push_back(ms);
    }
  }
  s->ran = true;
  s->reduced = true;
  s->layout = P.sweeps.back().perm;
  s->rank_sum_p.clear();
  return LRQ_OK;
}

// all ranks: `count` doubles from every rank (device buffer src), in rank order
int gather_doubles(lrq_state* s, const double* src_dev, int count, std::vector<double>& h) {
  if (s->group) {
    lrq_group* G = s->group;
    std::vector<double> mine((size_t)count);
    CUDA_TRY(cudaMemcpyAsync(mine.data(), src_dev, sizeof(double) * count, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    {
      std::lock_guard<std::mutex> lk(G->mu);
      if (G->gather.size() < (size_t)count * G->world) G->gather.resize((size_t)count * G->world);
      memcpy(&G->gather[(size_t)count * s->rank], mine.data(), sizeof(double) * count);
    }
    int rc = group_barrier(G);
    if (rc) return rc;
    {
      std::lock_guard<std::mutex> lk(G->mu);
      h.assign(G->gather.begin(), G->gather.begin() + (size_t)count * G->world);
    }
    return group_barrier(G);  // nobody overwrites a slot before all have read
  }
  if (!s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
  NCCL_TRY_S(s, nccl().AllGather(src_dev, s->dgather, count, ncclDouble, s->comm, s->stream));
  h.resize((size_t)count * s->world);
  CUDA_TRY(cudaMemcpyAsync(h.data(), s->dgather, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s->stream));
  return dist_wait(s, s->stream);
}

// all ranks: the per-rank finalize scalars, gathered in rank order
int gather_out(lrq_state* s, std::vector<double>& h) {
  if (s->group) {
    lrq_group* G = s->group;
    double mine[kOutScalars];
    CUDA_TRY(cudaMemcpyAsync(mine, s->out, sizeof mine, cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    {
      std::lock_guard<std::mutex> lk(G->mu);
      memcpy(&G->gather[kOutScalars * s->rank], mine, sizeof mine);
    }
    int rc = group_barrier(G);
    if (rc) return rc;
    {
      std::lock_guard<std::mutex> lk(G->mu);
      h = G->gather;
    }
    return group_barrier(G);  // nobody overwrites a slot before all have read
  }
  if (!s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
  NCCL_TRY_S(s, nccl().AllGather(s->out, s->dgather, kOutScalars, ncclDouble, s->comm, s->stream));
  h.resize(kOutScalars * s->world);
  CUDA_TRY(cudaMemcpyAsync(h.data(), s->dgather, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s->stream));
  return dist_wait(s, s->stream);
}

}  // namespace

extern "C" {

int lrq_nccl_unique_id(void* out, size_t cap) {
  if (!out || cap < sizeof(ncclUniqueId)) return fail(LRQ_EVALIDATION, "unique-id buffer too small");
  NcclApi& nc = nccl();
  if (!nc.ok) return fail(LRQ_ERUNTIME, nc.err);
  ncclUniqueId id;
  NCCL_TRY(nc.GetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return LRQ_OK;
}

int lrq_dist_terms(int n, int g, int rank, int perm, const double* edges, double* mloc, double* ext,
                   double* cst) {
  if (n < 2 || g < 0 || g >= n || !edges || !mloc || !ext || !cst) return fail(LRQ_EVALIDATION, "bad argument");
  if (rank < 0 || rank >= (1 << g)) return fail(LRQ_EVALIDATION, "rank out of range");
  dist_terms(n, g, rank, perm, edges, mloc, ext, cst);
  return LRQ_OK;
}

int lrq_describe_dist_plan(int n, int g, int pbytes, int p, char* buf, size_t cap) {
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  if (g < 1 || g > 6) return fail(LRQ_EVALIDATION, "log2(world) out of range [1, 6]");
  if (p < 1) return fail(LRQ_EVALIDATION, "p must be >= 1");
  const int nl = n - g, KA = tile_amp_bits(pbytes);
  if (nl <= KA) return fail(LRQ_EVALIDATION, "distributed engine needs n - log2(world) > " + std::to_string(KA));
  const Plan P = make_dist_plan(nl, g, pair_of(pbytes), p);
  if (P.groups.back().ntargets < g)
    return fail(LRQ_EVALIDATION, "last qubit group smaller than log2(world); choose another n");
  std::string js = plan_json(P);
  // append the distributed fields per sweep: [perm, remap_after, target1]
  js.pop_back();
  js += ",\"dist\":[";
  for (size_t i = 0; i < P.sweeps.size(); ++i) {
    const PlanSweep& w = P.sweeps[i];
    js += (i ? "," : "");
    js += "[" + std::to_string(w.perm) + "," + (w.remap_after ? "1" : "0") + "," + std::to_string(w.target1) + "]";
  }
  js += "]}";
  if (!buf || cap < js.size() + 1) return fail(LRQ_EVALIDATION, "buffer too small: need " + std::to_string(js.size() + 1));
  memcpy(buf, js.c_str(), js.size() + 1);
  return LRQ_OK;
}

int lrq_abi_version(void) { return LRQ_ABI_VERSION; }

const char* lrq_last_error(void) { return g_err.c_str(); }

int lrq_device_count(int* count) {
  if (!count) return fail(LRQ_EVALIDATION, "null count");
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(LRQ_ERUNTIME, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  *count = c;
  return LRQ_OK;
}

int lrq_describe_remap(int world, int rank, int mirror, char* buf, size_t cap) {
  if (world < 2 || (world & (world - 1))) return fail(LRQ_EVALIDATION, "world size must be a power of two >= 2");
  if (rank < 0 || rank >= world || mirror >= world) return fail(LRQ_EVALIDATION, "rank out of range");
  std::string js = "[";
  const std::vector<RemapStep> v = remap_schedule(world, rank, mirror);
  for (size_t i = 0; i < v.size(); ++i)
    js += (i ? "," : "") + std::string("[") + std::to_string(v[i].partner) + "," + std::to_string(v[i].my_block) +
          "," + std::to_string(v[i].their_block) + "," + std::to_string(v[i].half) + "]";
  js += "]";
  if (!buf || cap < js.size() + 1) return fail(LRQ_EVALIDATION, "buffer too small: need " + std::to_string(js.size() + 1));
  memcpy(buf, js.c_str(), js.size() + 1);
  return LRQ_OK;
}

int lrq_describe_memory(int n, int pbytes, int world, int p, uint64_t* state_bytes, uint64_t* other_bytes,
                        uint64_t* extra_spare) {
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  if (world < 1 || (world & (world - 1))) return fail(LRQ_EVALIDATION, "world size must be a power of two");
  int g = 0;
  while ((1 << g) < world) ++g;
  if (n - g < 1 || n - g > 40) return fail(LRQ_EVALIDATION, "qubits per rank out of range [1, 40]");
  const int nl = n - g;
  const uint64_t st = (uint64_t)pbytes << nl;
  if (state_bytes) *state_bytes = st;
  if (other_bytes) *other_bytes = rank_extra_bytes(nl, pbytes, world, p, world > 1);
  if (extra_spare) *extra_spare = world > 1 ? st : 0;
  return LRQ_OK;
}

int lrq_describe_plan(int n, int pbytes, int p, char* buf, size_t cap) {
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  if (n < 1 || n > 40) return fail(LRQ_EVALIDATION, "num_qubits out of range [1, 40]");
  if (p < 1) return fail(LRQ_EVALIDATION, "p must be >= 1");
  const std::string js = plan_json(make_plan(n, pair_of(pbytes), p));
  if (!buf || cap < js.size() + 1) return fail(LRQ_EVALIDATION, "buffer too small: need " + std::to_string(js.size() + 1));
  memcpy(buf, js.c_str(), js.size() + 1);
  return LRQ_OK;
}

int lrq_create(int n, int pbytes, int device, uint64_t budget, lrq_state** out) {
  if (!out) return fail(LRQ_EVALIDATION, "null output handle");
  *out = nullptr;
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  if (n < 1) return fail(LRQ_EVALIDATION, "need at least one qubit, got " + std::to_string(n));
  if (n > 40) return fail(LRQ_ECAPACITY, "num_qubits > 40 is not supported on one device");
  const size_t need = (size_t)pbytes << n;
  const char* prec = pbytes == 8 ? "fp32" : "fp64";
  if (budget && need > budget)
    return fail(LRQ_ECAPACITY, "statevector for " + std::to_string(n) + " qubits at " + prec + " needs " +
                                   std::to_string(need) + " bytes (" + gib((double)need) + " GiB), budget is " +
                                   std::to_string(budget) + " bytes");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRQ_ERUNTIME, "no CUDA device available (the LR-QAOA engine has no CPU path)");
  if (device < 0 || device >= ndev) return fail(LRQ_EVALIDATION, "device index out of range");
  DeviceGuard guard(device);
  size_t freeb = 0, totalb = 0;
  CUDA_TRY(cudaMemGetInfo(&freeb, &totalb));
  if (need + (256ull << 20) > freeb)
    return fail(LRQ_ECAPACITY, "statevector for " + std::to_string(n) + " qubits at " + prec + " needs " +
                                   std::to_string(need) + " bytes (" + gib((double)need) +
                                   " GiB), device has " + std::to_string(freeb) + " bytes free");
  lrq_state* s = new lrq_state();
  s->n = n;
  s->pbytes = pbytes;
  s->device = device;
  s->K = tile_amp_bits(pbytes);
  s->state_bytes = need;
  s->num_tiles = n >= s->K ? (1ll << (n - s->K)) : 1;
  cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&s->amps, need);
  if (e == cudaSuccess) e = cudaMalloc(&s->red, sizeof(double) * kRedArrays * s->num_tiles);
  if (e == cudaSuccess) e = cudaMalloc(&s->prefix, sizeof(double) * (s->num_tiles + 1));
  if (e == cudaSuccess) e = cudaMalloc(&s->out, sizeof(double) * kOutScalars);
  if (e == cudaSuccess) e = cudaMalloc(&s->fin, sizeof(double) * kFinScratch);
  // zero-fills on the engine's own (non-blocking) stream and waited for: a
  // legacy-stream cudaMemset is not ordered with it and could land after the
  // first lrq_set_cost copy
  if (e == cudaSuccess) e = cudaMalloc(&s->dW, sizeof(double) * n * n);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dW, 0, sizeof(double) * n * n, s->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->dzero, sizeof(double) * (n + 1));
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dzero, 0, sizeof(double) * (n + 1), s->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) {
    free_state(s);
    return fail(e == cudaErrorMemoryAllocation ? LRQ_ECAPACITY : LRQ_ERUNTIME,
                std::string("device allocation failed: ") + cudaGetErrorString(e));
  }
  *out = s;
  return LRQ_OK;
}

int lrq_destroy(lrq_state* s) {
  free_state(s);
  return LRQ_OK;
}

namespace {
// common part of lrq_create_dist / lrq_create_shard: a rank's shard of
// 2^(n_total-g) amplitudes plus the remap / gather buffers
int create_rank_state(int n_total, int pbytes, int device, int rank, int world, uint64_t memory_budget,
                      bool staging, lrq_state** out) {
  if (world < 2 || (world & (world - 1))) return fail(LRQ_EVALIDATION, "world size must be a power of two >= 2");
  if (rank < 0 || rank >= world) return fail(LRQ_EVALIDATION, "rank out of range");
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  int g = 0;
  while ((1 << g) < world) ++g;
  const int nl = n_total - g, KA = tile_amp_bits(pbytes);
  if (nl <= KA) return fail(LRQ_EVALIDATION, "distributed engine needs n - log2(world) > " + std::to_string(KA));
  if (make_dist_plan(nl, g, pair_of(pbytes), 1).groups.back().ntargets < g)
    return fail(LRQ_EVALIDATION, "last qubit group smaller than log2(world); choose another n");
  lrq_state* s = nullptr;
  int rc = lrq_create(nl, pbytes, device, memory_budget, &s);
  if (rc) return rc;
  s->world = world;
  s->rank = rank;
  s->g = g;
  s->n_total = n_total;
  DeviceGuard guard(device);
  const size_t block = (size_t)pbytes << (nl - g);
  s->chunk = remap_chunk(block);
  s->bufs[0] = s->amps;  // the primary buffer; a fused-remap spare comes later (group_prepare / lrq_ipc_handles)
  cudaError_t e = staging ? cudaMalloc(&s->stage, s->chunk) : cudaSuccess;
  if (e == cudaSuccess) e = cudaMalloc(&s->dWx, sizeof(double) * nl);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dWx, 0, sizeof(double) * nl, s->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->dW1, sizeof(double) * nl * nl);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dW1, 0, sizeof(double) * nl * nl, s->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->dWx1, sizeof(double) * nl);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dWx1, 0, sizeof(double) * nl, s->stream);
  // all-gathered scalars: kOutScalars per rank, or world block masses per rank
  if (e == cudaSuccess) e = cudaMalloc(&s->dgather, sizeof(double) * (kOutScalars + world) * world);
  if (e == cudaSuccess) e = cudaMalloc(&s->dflag, 2 * sizeof(float));
  if (e == cudaSuccess) e = cudaMemsetAsync(s->dflag, 0, 2 * sizeof(float), s->stream);
  if (e == cudaSuccess) e = cudaMalloc(&s->probe, sizeof(float) * world);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) {
    free_state(s);
    return fail(LRQ_ECAPACITY, std::string("distributed buffers: ") + cudaGetErrorString(e));
  }
  *out = s;
  return LRQ_OK;
}
}  // namespace

int lrq_create_dist(int n_total, int pbytes, int device, int rank, int world, const void* nccl_id,
                    uint64_t memory_budget, lrq_state** out) {
  if (!out || !nccl_id) return fail(LRQ_EVALIDATION, "null argument");
  *out = nullptr;
  NcclApi& nc = nccl();
  if (!nc.ok) return fail(LRQ_ERUNTIME, nc.err);
  lrq_state* s = nullptr;
  int rc = create_rank_state(n_total, pbytes, device, rank, world, memory_budget, true, &s);
  if (rc) return rc;
  DeviceGuard guard(device);
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof id);
  ncclResult_t r = nc.CommInitRank(&s->comm, world, id, rank);
  if (r != ncclSuccess) {
    s->comm = nullptr;
    free_state(s);
    return fail(LRQ_ERUNTIME, std::string("ncclCommInitRank: ") + nc.GetErrorString(r));
  }
  *out = s;
  return LRQ_OK;
}

int lrq_ipc_handles(lrq_state* s, void* out, size_t cap) {
  if (!s || !out) return fail(LRQ_EVALIDATION, "null argument");
  if (cap < LRQ_IPC_HANDLE_BYTES) return fail(LRQ_EVALIDATION, "handle buffer too small");
  memset(out, 0, LRQ_IPC_HANDLE_BYTES);
  // zero handles: NCCL transport only ($LRQ_PEER_REMAP=0 forces it)
  if (s->world < 2 || s->world > 8 || s->group || !env_int("LRQ_PEER_REMAP", 1)) return LRQ_OK;
  DeviceGuard guard(s->device);
  // the fused remap's spare state buffer, only if it fits with 2 GiB to spare
  // (lrq_fused_setup frees it again unless every rank got one)
  if (!s->bufs[1] && env_int("LRQ_FUSED_REMAP", 1)) {
    size_t freeb = 0, totalb = 0;
    if (cudaMemGetInfo(&freeb, &totalb) == cudaSuccess && freeb >= s->state_bytes + (2ull << 30)) {
      void* alt = nullptr;
      if (cudaMalloc(&alt, s->state_bytes) == cudaSuccess) s->bufs[1] = alt;
    }
    cudaGetLastError();
  }
  cudaIpcMemHandle_t h[3];
  memset(h, 0, sizeof h);
  CUDA_TRY(cudaIpcGetMemHandle(&h[0], s->bufs[0]));
  if (s->bufs[1]) CUDA_TRY(cudaIpcGetMemHandle(&h[1], s->bufs[1]));
  CUDA_TRY(cudaIpcGetMemHandle(&h[2], s->probe));
  memcpy(out, h, sizeof h);
  return LRQ_OK;
}

// peer writes of the remap self-test: rank writes (rank + 1) into slot `rank`
// of every rank's probe buffer
__global__ void peer_probe_kernel(float* const* dst, int world, int rank) {
  const int b = threadIdx.x;
  if (b < world) dst[b][rank] = (float)(rank + 1);
}

int lrq_fused_setup(lrq_state* s, const void* all_handles, int* enabled) {
  if (!s || !all_handles || !enabled) return fail(LRQ_EVALIDATION, "null argument");
  *enabled = 0;
  if (s->world < 2 || s->group) return fail(LRQ_EVALIDATION, "lrq_fused_setup is for NCCL ranks");
  if (!s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
  DeviceGuard guard(s->device);
  const int W = s->world;
  static const cudaIpcMemHandle_t zero = {};
  auto handle = [&](int b, int i) {
    return reinterpret_cast<const cudaIpcMemHandle_t*>(static_cast<const unsigned char*>(all_handles) +
                                                       (size_t)b * LRQ_IPC_HANDLE_BYTES)[i];
  };
  // map the peers' primary buffers and probes (and spare buffers if all have one)
  bool peer = W <= 8, spare = W <= 8;
  std::vector<float*> probes(W, nullptr);
  for (int b = 0; b < W && peer; ++b) {
    if (b == s->rank) {
      s->peer[0][b] = s->bufs[0];
      s->peer[1][b] = s->bufs[1];
      probes[b] = s->probe;
      spare = spare && s->bufs[1];
      continue;
    }
    const cudaIpcMemHandle_t h0 = handle(b, 0), h1 = handle(b, 1), h2 = handle(b, 2);
    if (!memcmp(&h0, &zero, sizeof zero) || !memcmp(&h2, &zero, sizeof zero)) {
      peer = false;
      break;
    }
    void* p0 = nullptr;
    void* p2 = nullptr;
    if (cudaIpcOpenMemHandle(&p0, h0, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&p2, h2, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      if (p0) cudaIpcCloseMemHandle(p0);
      peer = false;
      break;
    }
    s->ipc_open.push_back(p0);
    s->ipc_open.push_back(p2);
    s->peer[0][b] = p0;
    probes[b] = reinterpret_cast<float*>(p2);
    spare = spare && memcmp(&h1, &zero, sizeof zero) != 0;
  }
  spare = spare && peer && s->bufs[1];
  std::vector<void*> spares;
  for (int b = 0; b < W && spare; ++b) {
    if (b == s->rank) continue;
    void* p1 = nullptr;
    if (cudaIpcOpenMemHandle(&p1, handle(b, 1), cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      spare = false;
      break;
    }
    spares.push_back(p1);
    s->peer[1][b] = p1;
  }
  // collective self-test of the peer stores (every rank takes part even if its
  // own mapping failed, so the collectives stay matched)
  float** dptr = nullptr;
  float* dv = nullptr;
  CUDA_TRY(cudaMalloc(&dptr, sizeof(float*) * W));
  CUDA_TRY(cudaMalloc(&dv, 2 * sizeof(float)));
  CUDA_TRY(cudaMemsetAsync(s->probe, 0, sizeof(float) * W, s->stream));
  CUDA_TRY(cudaMemcpyAsync(dptr, probes.data(), sizeof(float*) * W, cudaMemcpyHostToDevice, s->stream));
  int rc = dist_wait(s, s->stream);
  if (rc) return rc;
  NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, s->stream));  // probes zeroed
  if (peer) {
    peer_probe_kernel<<<1, 32, 0, s->stream>>>(dptr, W, s->rank);
    CUDA_TRY(cudaGetLastError());
  }
  NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, s->stream));  // probes written
  if ((rc = dist_wait(s, s->stream))) return rc;
  float good[2] = {peer ? 1.0f : 0.0f, spare ? 1.0f : 0.0f};
  if (peer) {
    std::vector<float> got(W);
    CUDA_TRY(cudaMemcpy(got.data(), s->probe, sizeof(float) * W, cudaMemcpyDeviceToHost));
    for (int b = 0; b < W; ++b)
      if (got[b] != (float)(b + 1)) good[0] = good[1] = 0.0f;
  }
  // enabled only if every rank passed: minimum over ranks
  CUDA_TRY(cudaMemcpy(dv, good, sizeof good, cudaMemcpyHostToDevice));
  NCCL_TRY_S(s, nccl().AllReduce(dv, dv, 2, ncclFloat, ncclMin, s->comm, s->stream));
  if ((rc = dist_wait(s, s->stream))) return rc;
  CUDA_TRY(cudaMemcpy(good, dv, sizeof good, cudaMemcpyDeviceToHost));
  cudaFree(dptr);
  cudaFree(dv);
  s->peer_ok = good[0] == 1.0f;
  s->fused = s->peer_ok && good[1] == 1.0f;
  if (!s->fused) {
    // no fused remap anywhere: drop the spare buffer and the peers' mappings of theirs
    for (void* q : spares) cudaIpcCloseMemHandle(q);
    for (int b = 0; b < 8; ++b) s->peer[1][b] = nullptr;
    if (s->bufs[1]) {
      CUDA_TRY(cudaStreamSynchronize(s->stream));
      // every rank has closed its mapping of our spare before we free it
      NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, s->stream));
      if ((rc = dist_wait(s, s->stream))) return rc;
      if (s->cur == 1) {
        CUDA_TRY(cudaMemcpy(s->bufs[0], s->bufs[1], s->state_bytes, cudaMemcpyDeviceToDevice));
        s->cur = 0;
        s->amps = s->bufs[0];
      }
      cudaFree(s->bufs[1]);
      s->bufs[1] = nullptr;
    } else {
      NCCL_TRY_S(s, nccl().AllReduce(s->dflag, s->dflag, 1, ncclFloat, ncclSum, s->comm, s->stream));
      if ((rc = dist_wait(s, s->stream))) return rc;
    }
  } else {
    for (void* q : spares) s->ipc_open.push_back(q);
  }
  *enabled = s->fused ? 1 : (s->peer_ok ? 2 : 0);
  return LRQ_OK;
}

int lrq_group_create(int world, lrq_group** out) {
  if (!out) return fail(LRQ_EVALIDATION, "null argument");
  *out = nullptr;
  if (world < 2 || (world & (world - 1))) return fail(LRQ_EVALIDATION, "world size must be a power of two >= 2");
  lrq_group* G = new lrq_group;
  G->world = world;
  G->members.assign(world, nullptr);
  G->gather.assign(kOutScalars * (size_t)world, 0.0);
  G->shot_bufs.assign(world, nullptr);
  *out = G;
  return LRQ_OK;
}

int lrq_group_abort(lrq_group* G) {
  if (!G) return fail(LRQ_EVALIDATION, "null group");
  group_abort(G, "aborted by the host");
  return LRQ_OK;
}

int lrq_group_destroy(lrq_group* G) {
  if (!G) return LRQ_OK;
  {
    std::lock_guard<std::mutex> lk(G->mu);
    for (lrq_state* m : G->members)
      if (m) return fail(LRQ_ERUNTIME, "destroy the group's shard states first");
  }
  delete G;
  return LRQ_OK;
}

int lrq_create_shard(int n_total, int pbytes, int device, int rank, lrq_group* G, uint64_t memory_budget,
                     lrq_state** out) {
  if (!out || !G) return fail(LRQ_EVALIDATION, "null argument");
  *out = nullptr;
  {
    std::lock_guard<std::mutex> lk(G->mu);
    if (rank < 0 || rank >= G->world) return fail(LRQ_EVALIDATION, "rank out of range");
    if (G->members[rank]) return fail(LRQ_EVALIDATION, "rank already has a shard in this group");
  }
  lrq_state* s = nullptr;
  int rc = create_rank_state(n_total, pbytes, device, rank, G->world, memory_budget, false, &s);
  if (rc) return rc;
  std::lock_guard<std::mutex> lk(G->mu);
  if (G->members[rank]) {
    free_state(s);
    return fail(LRQ_EVALIDATION, "rank already has a shard in this group");
  }
  s->group = G;
  G->members[rank] = s;
  *out = s;
  return LRQ_OK;
}

int lrq_dist_layout(lrq_state* s, int* layout_out) {
  if (!s || !layout_out) return fail(LRQ_EVALIDATION, "null argument");
  *layout_out = s->layout;
  return LRQ_OK;
}

int lrq_dist_info(lrq_state* s, int* n_local, int* rank, int* world) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (n_local) *n_local = s->n;
  if (rank) *rank = s->rank;
  if (world) *world = s->world;
  return LRQ_OK;
}

int lrq_set_cost(lrq_state* s, const double* w) {
  if (!s || !w) return fail(LRQ_EVALIDATION, "null argument");
  const int n = s->n, nt = s->world > 1 ? s->n_total : s->n, E = nt * (nt - 1) / 2;
  std::vector<double> M((size_t)n * n);
  double tot = 0.0;
  for (int e = 0; e < E; ++e) {
    if (!isfinite(w[e])) return fail(LRQ_EVALIDATION, "edge weight is not finite");
    tot += w[e];
  }
  DeviceGuard guard(s->device);
  if (s->world > 1) {
    // local view in the identity permutation (the final pass runs there)
    std::vector<double> ext(n), M1((size_t)n * n), ext1(n);
    s->cost_edges.assign(w, w + E);
    dist_terms(nt, s->g, s->rank, 0, w, M.data(), ext.data(), &s->wcst);
    dist_terms(nt, s->g, s->rank, 1, w, M1.data(), ext1.data(), &s->wcst1);
    CUDA_TRY(cudaMemcpyAsync(s->dWx, ext.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->dW1, M1.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaMemcpyAsync(s->dWx1, ext1.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
  } else {
    sym_matrix(n, w, M.data());
  }
  CUDA_TRY(cudaMemcpyAsync(s->dW, M.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->wtot = tot;
  s->have_cost = true;
  s->reduced = false;
  return LRQ_OK;
}

int lrq_run(lrq_state* s, int p, const double* phase, const double* mixer) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (p < 1) return fail(LRQ_EVALIDATION, "depth p must be >= 1");
  if (!phase || !mixer) return fail(LRQ_EVALIDATION, "null phase/mixer arrays");
  const int n = s->n, nt = s->world > 1 ? s->n_total : n, E = n * (n - 1) / 2, Et = nt * (nt - 1) / 2;
  for (long long i = 0; i < (long long)p * Et; ++i)
    if (!isfinite(phase[i])) return fail(LRQ_EVALIDATION, "phase angle is not finite");
  for (int k = 0; k < p; ++k)
    if (!isfinite(mixer[k])) return fail(LRQ_EVALIDATION, "mixer angle is not finite");
  DeviceGuard guard(s->device);
  NvtxRange nv_run(s->world > 1 ? "lrq_run (distributed)" : "lrq_run");
  if (s->world > 1) {
    const int rc = run_dist(s, p, phase, mixer);
    if (rc && s->group) group_abort(s->group, g_err);
    return rc;
  }
  if (p > s->jcap) {
    cudaFree(s->dJ);
    cudaFree(s->dmix);
    s->dJ = nullptr;
    s->dmix = nullptr;
    CUDA_TRY(cudaMalloc(&s->dJ, sizeof(double) * (size_t)p * n * n));
    CUDA_TRY(cudaMalloc(&s->dmix, sizeof(double) * 2 * p));
    s->jcap = p;
  }
  std::vector<double> J((size_t)p * n * n), mix(2 * p);
  for (int k = 0; k < p; ++k) {
    sym_matrix(n, phase + (size_t)k * E, J.data() + (size_t)k * n * n);
    mix[2 * k] = cos(mixer[k]);
    mix[2 * k + 1] = -sin(mixer[k]);
  }
  CUDA_TRY(cudaMemcpyAsync(s->dJ, J.data(), sizeof(double) * J.size(), cudaMemcpyHostToDevice, s->stream));
  CUDA_TRY(cudaMemcpyAsync(s->dmix, mix.data(), sizeof(double) * mix.size(), cudaMemcpyHostToDevice, s->stream));
  const bool fields = !s->field_h.empty();
  if (fields) {
    if (p > s->fcap) {
      cudaFree(s->dF);
      s->dF = nullptr;
      CUDA_TRY(cudaMalloc(&s->dF, sizeof(double) * (size_t)p * (n + 1)));
      s->fcap = p;
    }
    // The sweep path defers the X^(x)n of flipped mixers (mixer_form): after
    // an odd number of them the stored state is the index-reversed one, on
    // which Z_i reads -Z_i.  Z-Z terms are invariant; single-Z fields flip.
    std::vector<double> F(s->field_h);
    F.insert(F.end(), s->cst_h.begin(), s->cst_h.end());
    if (n >= s->K) {
      int fl = 0;
      for (int k = 0; k < p; ++k) {
        if (fl & 1)
          for (int i = 0; i < n; ++i) F[(size_t)k * n + i] = -F[(size_t)k * n + i];
        fl += mixer_form(mixer[k]).flip;
      }
    }
    CUDA_TRY(cudaMemcpyAsync(s->dF, F.data(), sizeof(double) * F.size(), cudaMemcpyHostToDevice, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));  // F is a local
  }

  const double init = s->pbytes == 8 ? init_amplitude<float>(n) : init_amplitude<double>(n);
  s->reduced = false;
  s->ran = false;
  s->kinds.clear();
  size_t ev = 0;
  record(s, ev++, 0);
  double* rp = s->red;
  double* rpe = rp + s->num_tiles;
  double* rmin = rpe + s->num_tiles;
  unsigned long long* rarg = reinterpret_cast<unsigned long long*>(rmin + s->num_tiles);
  double* rmax = rmin + 2 * s->num_tiles;
  const int min_bit = n - 1;

  if (n < s->K) {
    SmallParams sp;
    memset(&sp, 0, sizeof sp);
    sp.amps = s->amps;
    sp.n = n;
    sp.p = p;
    sp.J = s->dJ;
    sp.mix = s->dmix;
    sp.W = s->dW;  // zero until a cost is set: sum p is still reduced
    sp.F = fields ? s->dF : nullptr;
    sp.Fc = fields ? s->dF + (size_t)p * n : nullptr;
    if (!s->msign_h.empty()) {
      if (s->msign_h.size() > s->msign_cap) {
        cudaFree(s->dmsign);
        s->dmsign = nullptr;
        CUDA_TRY(cudaMalloc(&s->dmsign, s->msign_h.size()));
        s->msign_cap = s->msign_h.size();
      }
      CUDA_TRY(cudaMemcpyAsync(s->dmsign, s->msign_h.data(), s->msign_h.size(), cudaMemcpyHostToDevice, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
      sp.msign = s->dmsign;
    }
    sp.init_re = init;
    sp.init_im = 0.0;
    sp.load = 0;
    sp.min_bit = min_bit;
    sp.red_p = rp;
    sp.red_pE = rpe;
    sp.red_minE = rmin;
    sp.red_arg = rarg;
    sp.red_maxE = rmax;
    if (const int rh = zero_hist(s)) return rh;
    set_hist(s, sp);
    int rc = launch_small_any(s->pbytes, sp, s->stream);
    if (rc) return rc;
    record(s, ev++, 'S');
  } else {
    const Plan P = make_plan(n, pair_of(s->pbytes), p);
    const int grid_cap = 2 * sm_count(s->device);
    const int grid = (int)(s->num_tiles < grid_cap ? s->num_tiles : grid_cap);
    for (const PlanSweep& w : P.sweeps) {
      const PlanGroup& g = P.groups[w.group];
      SweepParams sp;
      memset(&sp, 0, sizeof sp);
      sp.amps = s->amps;
      sp.n = n;
      sp.q0 = g.q0;
      sp.num_tiles = s->num_tiles;
      sp.reduce = w.reduce ? 1 : 0;
      double sre = 1.0, sim = 0.0;
      const bool signed_mix = !s->msign_h.empty();
      if (w.beta1 >= 0) {
        const MixerForm f = mixer_form(mixer[w.beta1]);
        int neg = 0;
        if (signed_mix)
          neg = fill_tangents_signed(sp, 0, g, w, pair_of(s->pbytes), w.mask1, f.t, &s->msign_h[(size_t)w.beta1 * n]);
        else
          fill_tangents(sp, 0, w.mask1, w.nrounds, f.t);
        cpow_mul(sre, sim, f.qre, f.qim, g.ntargets);
        if (f.flip && (neg & 1)) sre = -sre, sim = -sim;  // (i s) per qubit: odd sign
      }
      if (w.beta2 >= 0) {
        const MixerForm f = mixer_form(mixer[w.beta2]);
        int neg = 0;
        if (signed_mix)
          neg = fill_tangents_signed(sp, 1, g, w, pair_of(s->pbytes), w.mask2, f.t, &s->msign_h[(size_t)w.beta2 * n]);
        else
          fill_tangents(sp, 1, w.mask2, w.nrounds, f.t);
        cpow_mul(sre, sim, f.qre, f.qim, g.ntargets);
        if (f.flip && (neg & 1)) sre = -sre, sim = -sim;
      }
      if (g.cross >= 0) {
        // the cross qubit of a cluster group: its tangents, and its sign in
        // the (i s)^k factor of a flipped layer with per-qubit signs
        for (int m = 0; m < 2; ++m) {
          const int b = m == 0 ? w.beta1 : w.beta2;
          sp.tc[m] = 0.0;
          if (b < 0) continue;
          const MixerForm f = mixer_form(mixer[b]);
          const bool negq = signed_mix && s->msign_h[(size_t)b * n + g.cross] < 0;
          sp.tc[m] = negq ? -f.t : f.t;
          if (f.flip && negq) sre = -sre, sim = -sim;
        }
      }
      sp.scale_re = sre;
      sp.scale_im = sim;
      sp.init_re = init;
      sp.init_im = 0.0;
      sp.J.M = w.phase >= 0 ? s->dJ + (size_t)w.phase * n * n : s->dW;
      sp.J.ext = fields && w.phase >= 0 ? s->dF + (size_t)w.phase * n : s->dzero;
      sp.J.cst = fields && w.phase >= 0 ? s->cst_h[w.phase] : 0.0;
      sp.W.M = s->dW;
      sp.W.ext = s->dzero;
      sp.W.cst = 0.0;
      sp.min_bit = min_bit;
      sp.red_p = rp;
      sp.red_pE = rpe;
      sp.red_minE = rmin;
      sp.red_arg = rarg;
      sp.red_maxE = rmax;
      if (w.reduce) {
        if (const int rh = zero_hist(s)) return rh;
        set_hist(s, sp);
      }
      char kname[2] = {"PMFRLQN"[w.kind], 0};
      NvtxRange nv_sweep(kname, group_name(g.kind));
      int rc = w.prog == 2   ? launch_wdc(s, g.kind, w.kind, sp)
               : w.prog == 1 ? launch_wd(s, g.kind, w.kind, sp)
                             : launch_sweep(s, g.kind, w.kind, sp, grid);
      if (rc) return rc;
      record(s, ev++, "PMFRLQN"[w.kind]);
    }
    int flips = 0;
    for (int k = 0; k < p; ++k) flips += mixer_form(mixer[k]).flip;
    if (flips & 1) {
      // deferred X^(x)n of the flipped layers: reverse the index order once;
      // tile b of the CDF becomes tile T-1-b (E and the max-cut are invariant)
      const long long half = (1ll << n) / 2;
      const unsigned blocks = (unsigned)((half + 255) / 256);
      if (s->pbytes == 8) reverse_kernel<float2><<<blocks, 256, 0, s->stream>>>(s->amps, n);
      else reverse_kernel<double2><<<blocks, 256, 0, s->stream>>>(s->amps, n);
      CUDA_TRY(cudaGetLastError());
      reverse_kernel<double><<<(unsigned)((s->num_tiles / 2 + 255) / 256 + 1), 256, 0, s->stream>>>(
          rp, 63 - __builtin_clzll((unsigned long long)s->num_tiles));
      CUDA_TRY(cudaGetLastError());
      record(s, ev++, 'X');
    }
  }
  {
    const int rc = launch_finalize(s->stream, s->num_tiles, s->red, s->prefix, s->out, s->fin);
    if (rc) return rc;
  }
  record(s, ev++, 'Z');
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (s->timing) {
    s->last_ms.clear();
    for (size_t i = 1; i < ev; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, s->evs[i - 1], s->evs[i]);
      s->last_ms.push_back(ms);
    }
  }
  s->ran = true;
  s->reduced = true;
  return LRQ_OK;
}

int lrq_run_fields(lrq_state* s, int p, const double* phase, const double* field, const double* constant,
                   const double* mixer) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world > 1) return fail(LRQ_EVALIDATION, "lrq_run_fields is single-GPU only");
  if (p < 1) return fail(LRQ_EVALIDATION, "depth p must be >= 1");
  if (!field || !constant) return fail(LRQ_EVALIDATION, "null field/constant arrays");
  const int n = s->n;
  for (long long i = 0; i < (long long)p * n; ++i)
    if (!isfinite(field[i])) return fail(LRQ_EVALIDATION, "field angle is not finite");
  for (int k = 0; k < p; ++k)
    if (!isfinite(constant[k])) return fail(LRQ_EVALIDATION, "constant phase is not finite");
  s->field_h.assign(field, field + (size_t)p * n);
  s->cst_h.assign(constant, constant + p);
  const int rc = lrq_run(s, p, phase, mixer);
  s->field_h.clear();
  s->cst_h.clear();
  return rc;
}

int lrq_run_ex(lrq_state* s, int p, const double* phase, const double* mixer_q) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world > 1) return fail(LRQ_EVALIDATION, "lrq_run_ex is single-GPU only");
  if (p < 1 || !mixer_q) return fail(LRQ_EVALIDATION, "need p >= 1 and per-qubit mixer angles");
  const int n = s->n;
  std::vector<double> layer(p);
  s->msign_h.assign((size_t)p * n, 1);
  for (int k = 0; k < p; ++k) {
    layer[k] = mixer_q[(size_t)k * n];
    for (int q = 0; q < n; ++q) {
      const double h = mixer_q[(size_t)k * n + q];
      if (!isfinite(h) || fabs(h) != fabs(layer[k])) {
        s->msign_h.clear();
        return fail(LRQ_EVALIDATION, "per-qubit mixer angles of a layer must agree up to sign");
      }
      s->msign_h[(size_t)k * n + q] = (h == layer[k]) ? 1 : -1;
    }
  }
  const int rc = lrq_run(s, p, phase, layer.data());
  s->msign_h.clear();
  return rc;
}

// z <-> z ^ mask (a Pauli-X string on the mask's qubits, up to phase)
int lrq_permute_xor(lrq_state* s, uint64_t mask) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world > 1) return fail(LRQ_EVALIDATION, "lrq_permute_xor is single-GPU only");
  if (mask >> s->n) return fail(LRQ_EVALIDATION, "mask has bits above the state's qubits");
  if (!mask) return LRQ_OK;
  DeviceGuard guard(s->device);
  const int grid = 4 * sm_count(s->device);
  if (s->pbytes == 8) xor_permute_kernel<float2><<<grid, 256, 0, s->stream>>>(s->amps, s->n, mask);
  else xor_permute_kernel<double2><<<grid, 256, 0, s->stream>>>(s->amps, s->n, mask);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->reduced = false;
  return LRQ_OK;
}

int lrq_reset(lrq_state* s, int which) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world > 1) return fail(LRQ_EVALIDATION, "gate-by-gate execution is single-GPU");
  if (which != 0 && which != 1) return fail(LRQ_EVALIDATION, "reset: 0 = |0...0>, 1 = uniform");
  DeviceGuard guard(s->device);
  const int grid = 4 * sm_count(s->device);
  if (s->pbytes == 8) {
    const float v = (float)(1.0 / sqrt((double)(1ull << s->n)));
    reset_kernel<float><<<grid, 256, 0, s->stream>>>(s->amps, s->n, which, v);
  } else {
    const double v = 1.0 / sqrt((double)(1ull << s->n));
    reset_kernel<double><<<grid, 256, 0, s->stream>>>(s->amps, s->n, which, v);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->ran = true;
  s->reduced = false;
  return LRQ_OK;
}

int lrq_apply_gate(lrq_state* s, int kind, int q0, int q1, double theta) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world > 1) return fail(LRQ_EVALIDATION, "gate-by-gate execution is single-GPU");
  const int n = s->n;
  if (q0 < 0 || q0 >= n || (kind == 2 && (q1 < 0 || q1 >= n)))
    return fail(LRQ_EVALIDATION, "qubit out of range for " + std::to_string(n) + " qubits");
  if (kind == 2 && q0 == q1) return fail(LRQ_EVALIDATION, "RZZ qubits must differ");
  if (kind < 0 || kind > 5) return fail(LRQ_EVALIDATION, "gate kind: 0 H, 1 RX, 2 RZZ, 3 X, 4 Y, 5 Z");
  if ((kind == 1 || kind == 2) && !isfinite(theta)) return fail(LRQ_EVALIDATION, "gate angle is not finite");
  DeviceGuard guard(s->device);
  const int grid = 4 * sm_count(s->device);
  const bool f32 = s->pbytes == 8;
  if (kind == 2) {
    const double er = cos(-0.5 * theta), ei = sin(-0.5 * theta), dr = cos(0.5 * theta), di = sin(0.5 * theta);
    if (f32)
      rzz_kernel<float><<<grid, 256, 0, s->stream>>>(s->amps, n, q0, q1, (float)er, (float)ei, (float)dr, (float)di);
    else
      rzz_kernel<double><<<grid, 256, 0, s->stream>>>(s->amps, n, q0, q1, er, ei, dr, di);
  } else {
    const double c = kind == 0 ? 1.0 / sqrt(2.0) : cos(0.5 * theta), sn = kind == 0 ? 0.0 : sin(0.5 * theta);
    if (f32)
      gate1q_kernel<float><<<grid, 256, 0, s->stream>>>(s->amps, n, q0, kind, (float)c, (float)sn);
    else
      gate1q_kernel<double><<<grid, 256, 0, s->stream>>>(s->amps, n, q0, kind, c, sn);
  }
  CUDA_TRY(cudaGetLastError());
  s->ran = true;
  s->reduced = false;
  return LRQ_OK;
}

int lrq_noisy_batch(int n, int pbytes, int device, int trajectories, int p, const double* phase,
                    const double* mixer, const unsigned* xmask, int64_t shots, const double* u, double* probs_out,
                    uint64_t* idx_out) {
  if (pbytes != 8 && pbytes != 16) return fail(LRQ_EVALIDATION, "precision_bytes must be 8 or 16");
  const int K = tile_amp_bits(pbytes);
  if (n < 1 || n >= K)
    return fail(LRQ_EVALIDATION, "batched trajectories need 1 <= n < " + std::to_string(K) + " (use lrq_run_ex above)");
  if (trajectories < 1 || p < 1) return fail(LRQ_EVALIDATION, "need at least one trajectory and one layer");
  if (!phase || !mixer || (shots > 0 && (!u || !idx_out))) return fail(LRQ_EVALIDATION, "null argument");
  const int E = n * (n - 1) / 2, N = 1 << n;
  // per layer the mixer half-angles may differ only in sign across qubits and trajectories
  std::vector<double> mix(2 * (size_t)p);
  std::vector<signed char> sg((size_t)trajectories * p * n);
  for (int k = 0; k < p; ++k) {
    const double h0 = fabs(mixer[(size_t)k * n]);
    mix[2 * k] = cos(h0);
    mix[2 * k + 1] = -sin(h0);
    for (int t = 0; t < trajectories; ++t)
      for (int q = 0; q < n; ++q) {
        const double h = mixer[((size_t)t * p + k) * n + q];
        if (!isfinite(h) || fabs(h) != h0)
          return fail(LRQ_EVALIDATION, "per-qubit mixer angles of a layer must agree up to sign");
        sg[((size_t)t * p + k) * n + q] = h < 0 ? -1 : 1;
      }
  }
  std::vector<double> J((size_t)trajectories * p * n * n);
  for (long long i = 0; i < (long long)trajectories * p; ++i) {
    for (int e = 0; e < E; ++e)
      if (!isfinite(phase[i * E + e])) return fail(LRQ_EVALIDATION, "phase angle is not finite");
    sym_matrix(n, phase + i * E, J.data() + (size_t)i * n * n);
  }
  DeviceGuard guard(device);
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  double *dJ = nullptr, *dmix = nullptr, *dprobs = nullptr, *du = nullptr;
  signed char* dsg = nullptr;
  unsigned* dmask = nullptr;
  unsigned long long* didx = nullptr;
  cudaError_t e = cudaMalloc(&dJ, sizeof(double) * J.size());
  if (e == cudaSuccess) e = cudaMalloc(&dmix, sizeof(double) * mix.size());
  if (e == cudaSuccess) e = cudaMalloc(&dsg, sg.size());
  if (e == cudaSuccess) e = cudaMalloc(&dmask, sizeof(unsigned) * trajectories);
  if (e == cudaSuccess) e = cudaMalloc(&dprobs, sizeof(double) * (size_t)trajectories * N);
  if (e == cudaSuccess && shots > 0) e = cudaMalloc(&du, sizeof(double) * (size_t)trajectories * shots);
  if (e == cudaSuccess && shots > 0) e = cudaMalloc(&didx, sizeof(unsigned long long) * (size_t)trajectories * shots);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dJ, J.data(), sizeof(double) * J.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dmix, mix.data(), sizeof(double) * mix.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dsg, sg.data(), sg.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    if (xmask) e = cudaMemcpyAsync(dmask, xmask, sizeof(unsigned) * trajectories, cudaMemcpyHostToDevice, st);
    else e = cudaMemsetAsync(dmask, 0, sizeof(unsigned) * trajectories, st);
  }
  if (e == cudaSuccess && shots > 0)
    e = cudaMemcpyAsync(du, u, sizeof(double) * (size_t)trajectories * shots, cudaMemcpyHostToDevice, st);
  int rc = LRQ_OK;
  if (e == cudaSuccess) {
    SmallParams sp;
    memset(&sp, 0, sizeof sp);
    sp.n = n;
    sp.p = p;
    sp.J = dJ;
    sp.strideJ = (long long)p * n * n;
    sp.mix = dmix;
    sp.msign = dsg;
    sp.xmask = dmask;
    sp.probs = dprobs;
    sp.init_re = pbytes == 8 ? init_amplitude<float>(n) : init_amplitude<double>(n);
    sp.min_bit = -2;
    const size_t smem = (size_t)pbytes * N + 8 * 5 * 8;
    if (pbytes == 8) {
      rc = launch_small<float>(sp, smem, st, trajectories);
    } else {
      rc = launch_small<double>(sp, smem, st, trajectories);
    }
    if (!rc && shots > 0) {
      batch_sample_kernel<<<trajectories, 256, sizeof(double) * N, st>>>(dprobs, N, du, shots, didx);
      e = cudaGetLastError();
    }
  }
  if (!rc && e == cudaSuccess && probs_out)
    e = cudaMemcpyAsync(probs_out, dprobs, sizeof(double) * (size_t)trajectories * N, cudaMemcpyDeviceToHost, st);
  if (!rc && e == cudaSuccess && shots > 0)
    e = cudaMemcpyAsync(idx_out, didx, sizeof(uint64_t) * (size_t)trajectories * shots, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dJ);
  cudaFree(dmix);
  cudaFree(dsg);
  cudaFree(dmask);
  cudaFree(dprobs);
  cudaFree(du);
  cudaFree(didx);
  cudaStreamDestroy(st);
  if (rc) return rc;
  CUDA_TRY(e);
  return LRQ_OK;
}

int lrq_recompute(lrq_state* s) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  NvtxRange nv("lrq_recompute");
  if (!s->ran) return fail(LRQ_ERUNTIME, "state holds no circuit result yet");
  DeviceGuard guard(s->device);
  const int n = s->n;
  double* rp = s->red;
  double* rpe = rp + s->num_tiles;
  double* rmin = rpe + s->num_tiles;
  unsigned long long* rarg = reinterpret_cast<unsigned long long*>(rmin + s->num_tiles);
  double* rmax = rmin + 2 * s->num_tiles;
  if (n < s->K) {
    SmallParams sp;
    memset(&sp, 0, sizeof sp);
    sp.amps = s->amps;
    sp.n = n;
    sp.p = 0;
    sp.J = s->dW;
    sp.mix = s->dzero;
    sp.W = s->dW;
    sp.load = 1;
    sp.min_bit = n - 1;
    sp.red_p = rp;
    sp.red_pE = rpe;
    sp.red_minE = rmin;
    sp.red_arg = rarg;
    sp.red_maxE = rmax;
    if (const int rh = zero_hist(s)) return rh;
    set_hist(s, sp);
    int rc = launch_small_any(s->pbytes, sp, s->stream);
    if (rc) return rc;
  } else {
    SweepParams sp;
    memset(&sp, 0, sizeof sp);
    sp.amps = s->amps;
    sp.n = n;
    sp.q0 = s->K;
    sp.num_tiles = s->num_tiles;
    sp.reduce = 1;
    sp.scale_re = 1.0;
    sp.J.M = s->dW;
    sp.J.ext = s->dzero;
    // a shard: the rank's cost view in the layout the state is in, and the
    // max-cut search over global top bit 0
    if (s->world > 1) {
      sp.W = cost_view(s, s->layout);
      sp.min_bit = search_bit(s, s->layout);
    } else {
      sp.W.M = s->dW;
      sp.W.ext = s->dzero;
      sp.W.cst = 0.0;
      sp.min_bit = n - 1;
    }
    sp.red_p = rp;
    sp.red_pE = rpe;
    sp.red_minE = rmin;
    sp.red_arg = rarg;
    sp.red_maxE = rmax;
    if (const int rh = zero_hist(s)) return rh;
    set_hist(s, sp);
    const int grid_cap = 2 * sm_count(s->device);
    int rc = launch_sweep(s, GK_A, SK_Q, sp, (int)(s->num_tiles < grid_cap ? s->num_tiles : grid_cap));
    if (rc) return rc;
  }
  {
    const int rc = launch_finalize(s->stream, s->num_tiles, s->red, s->prefix, s->out, s->fin);
    if (rc) return rc;
  }
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->reduced = true;
  s->rank_sum_p.clear();
  return LRQ_OK;
}

int lrq_reduce(lrq_state* s, lrq_reduction* out) {
  if (!s || !out) return fail(LRQ_EVALIDATION, "null argument");
  if (!s->reduced) return fail(LRQ_ERUNTIME, "no reductions: set a cost and run the circuit first");
  DeviceGuard guard(s->device);
  double h[kOutScalars];
  if (s->world > 1) {
    // collective: every rank's scalars, combined in rank order (deterministic);
    // local argmin -> global index (rank bits on top, identity permutation)
    std::vector<double> all;
    int rc = gather_out(s, all);
    if (rc) {
      if (s->group) group_abort(s->group, g_err);
      return rc;
    }
    double sp = 0.0, spe = 0.0, mn = __builtin_inf(), mx = -__builtin_inf();
    uint64_t best = ~0ull;
    s->rank_sum_p.assign(s->world, 0.0);
    for (int r = 0; r < s->world; ++r) {
      const double* a = &all[kOutScalars * r];
      sp += a[0];
      spe += a[1];
      s->rank_sum_p[r] = a[0];
      mx = fmax(mx, a[4]);
      uint64_t z;
      memcpy(&z, &a[3], 8);
      if (z == ~0ull) continue;
      const uint64_t gz = global_index(s->n, s->g, r, s->layout, z);
      if (a[2] < mn || (a[2] == mn && gz < best)) {
        mn = a[2];
        best = gz;
      }
    }
    out->sum_p = sp;
    out->sum_p_cut = 0.5 * (s->wtot * sp - spe);
    out->min_energy = mn;
    out->argmax_cut = best;
    out->max_energy = mx;
    return LRQ_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(h, s->out, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  out->sum_p = h[0];
  out->sum_p_cut = 0.5 * (s->wtot * h[0] - h[1]);
  out->min_energy = h[2];
  uint64_t z;
  memcpy(&z, &h[3], 8);
  out->argmax_cut = z;
  out->max_energy = h[4];
  return LRQ_OK;
}

int lrq_restore_layout(lrq_state* s);

int lrq_sample(lrq_state* s, const double* u, int64_t shots, uint64_t* idx) {
  if (!s || !u || !idx) return fail(LRQ_EVALIDATION, "null argument");
  if (shots < 1) return fail(LRQ_EVALIDATION, "shot count must be positive, got " + std::to_string(shots));
  if (!s->reduced) return fail(LRQ_ERUNTIME, "no CDF: set a cost and run the circuit first");
  DeviceGuard guard(s->device);
  NvtxRange nv("lrq_sample");
  if (shots > s->shot_cap) {
    cudaFree(s->du);
    cudaFree(s->didx);
    s->du = nullptr;
    s->didx = nullptr;
    CUDA_TRY(cudaMalloc(&s->du, sizeof(double) * shots));
    CUDA_TRY(cudaMalloc(&s->didx, sizeof(unsigned long long) * shots));
    s->shot_cap = shots;
  }
  const int tile_bits = s->n < s->K ? s->n : s->K;
  const long long grid = (shots * 32 + 255) / 256;
  // one contiguous segment of the global CDF: tiles [t0, t0 + T) of this
  // state starting at global cumulative mass goff, global indices base + local
  auto segment = [&](long long t0, long long T, double goff, double total, unsigned long long base,
                     int write_unowned) {
    const void* amps = static_cast<const char*>(s->amps) + ((size_t)t0 << tile_bits) * s->pbytes;
    if (s->pbytes == 8)
      sample_kernel<float><<<(unsigned)grid, 256, 0, s->stream>>>(amps, tile_bits, T, s->prefix + t0, s->du, shots,
                                                                  goff, total, base, write_unowned, s->didx);
    else
      sample_kernel<double><<<(unsigned)grid, 256, 0, s->stream>>>(amps, tile_bits, T, s->prefix + t0, s->du, shots,
                                                                   goff, total, base, write_unowned, s->didx);
    return cudaGetLastError();
  };
  if (s->world > 1 && s->layout == 1 && (s->num_tiles >> s->g) == 0) {
    // blocks smaller than a tile (tiny shards): no per-block masses in the
    // tile prefix; make the remaining remap (collective, like this call)
    const int rc = lrq_restore_layout(s);
    if (rc) return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(s->du, u, sizeof(double) * shots, cudaMemcpyHostToDevice, s->stream));
  if (s->world > 1 && s->layout == 1) {
    // swapped layout: global index order visits block b (top g local bits) of
    // every rank in rank order, then block b+1: the CDF has world x world
    // segments; each rank owns `world` of them.  The block masses come from
    // the tile prefix, all-gathered; the uniforms in a segment are resolved
    // by its owner and an integer sum gives every rank all indices.
    const int G = s->world, g = s->g, nl = s->n;
    const long long TB = s->num_tiles >> g;
    std::vector<double> pre(G + 1);
    for (int b = 0; b <= G; ++b)
      CUDA_TRY(cudaMemcpyAsync(&pre[b], s->prefix + (size_t)b * TB, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    std::vector<double> mass(G);
    for (int b = 0; b < G; ++b) mass[b] = pre[b + 1] - pre[b];
    CUDA_TRY(cudaMemcpyAsync(s->dgather + (size_t)(kOutScalars + G) * G - G, mass.data(), sizeof(double) * G,
                             cudaMemcpyHostToDevice, s->stream));
    std::vector<double> all;  // all[r * G + b]
    int rc = gather_doubles(s, s->dgather + (size_t)(kOutScalars + G) * G - G, G, all);
    if (rc) {
      if (s->group) group_abort(s->group, g_err);
      return rc;
    }
    double total = 0.0;
    for (int b = 0; b < G; ++b)
      for (int r = 0; r < G; ++r) total += all[(size_t)r * G + b];
    if (!(total > 0.0)) return fail(LRQ_EVALIDATION, "statevector has zero norm, nothing to sample");
    CUDA_TRY(cudaMemsetAsync(s->didx, 0, sizeof(unsigned long long) * shots, s->stream));
    double off = 0.0;
    for (int b = 0; b < G; ++b)
      for (int r = 0; r < G; ++r) {
        if (r == s->rank) {
          const unsigned long long base = ((unsigned long long)b << nl) | ((unsigned long long)r << (nl - g));
          CUDA_TRY(segment((long long)b * TB, TB, off - pre[b], total, base, 0));
        }
        off += all[(size_t)r * G + b];
      }
  } else {
    double total = 0.0, off = 0.0;
    unsigned long long base_index = 0;
    if (s->world > 1) {
      // global CDF over ranks in rank order: this rank owns the uniforms that
      // land in [off, off + its mass) / total
      if ((int)s->rank_sum_p.size() != s->world) {
        lrq_reduction tmp;
        int rc = lrq_reduce(s, &tmp);
        if (rc) return rc;
      }
      for (int r = 0; r < s->world; ++r) {
        if (r == s->rank) off = total;
        total += s->rank_sum_p[r];
      }
      base_index = (unsigned long long)s->rank << s->n;
    } else {
      CUDA_TRY(cudaMemcpyAsync(&total, s->out, sizeof(double), cudaMemcpyDeviceToHost, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
    if (!(total > 0.0)) return fail(LRQ_EVALIDATION, "statevector has zero norm, nothing to sample");
    CUDA_TRY(segment(0, s->num_tiles, off, total, base_index, 1));
  }
  if (s->world > 1 && !s->group) {  // exactly one rank owns each shot; the others hold 0
    if (!s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
    NCCL_TRY_S(s, nccl().AllReduce(s->didx, s->didx, shots, ncclUint64, ncclSum, s->comm, s->stream));
  }
  CUDA_TRY(cudaMemcpyAsync(idx, s->didx, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, s->stream));
  if (s->world > 1 && !s->group) {
    const int rc = dist_wait(s, s->stream);
    if (rc) return rc;
  } else {
    CUDA_TRY(cudaStreamSynchronize(s->stream));
  }
  if (s->group) {
    const int rc = group_sum_shots(s, idx, shots);
    if (rc) group_abort(s->group, g_err);
    return rc;
  }
  return LRQ_OK;
}

// the identity layout back after an odd-p run (the one remap the run did not
// make); collective.  The reductions are recomputed in the new layout.
int lrq_restore_layout(lrq_state* s) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (s->world < 2 || s->layout == 0) return LRQ_OK;
  DeviceGuard guard(s->device);
  NvtxRange nv("lrq_restore_layout");
  int rc = remap_exchange(s, false, -1);
  if (rc) {
    if (s->group) group_abort(s->group, g_err);
    return rc;
  }
  s->layout = 0;
  if (s->reduced) return lrq_recompute(s);
  return LRQ_OK;
}

int lrq_store_amps(lrq_state* s, uint64_t start, uint64_t count, const void* host) {
  if (!s || (!host && count)) return fail(LRQ_EVALIDATION, "null argument");
  if (start + count > (1ull << s->n)) return fail(LRQ_EVALIDATION, "amplitude range out of bounds");
  s->layout = 0;  // the caller writes identity-layout amplitudes
  DeviceGuard guard(s->device);
  CUDA_TRY(cudaMemcpyAsync((char*)s->amps + start * s->pbytes, host, count * s->pbytes, cudaMemcpyHostToDevice,
                           s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->ran = true;
  s->reduced = false;
  return LRQ_OK;
}

int lrq_copy_amps(lrq_state* s, uint64_t start, uint64_t count, void* host) {
  if (!s || (!host && count)) return fail(LRQ_EVALIDATION, "null argument");
  if (start + count > (1ull << s->n)) return fail(LRQ_EVALIDATION, "amplitude range out of bounds");
  if (s->layout != 0)
    return fail(LRQ_ERUNTIME, "the shard is in the swapped layout of an odd-p run: call lrq_restore_layout (collective) first");
  DeviceGuard guard(s->device);
  CUDA_TRY(cudaMemcpyAsync(host, (const char*)s->amps + start * s->pbytes, count * s->pbytes, cudaMemcpyDeviceToHost,
                           s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return LRQ_OK;
}

int lrq_cut_values(int n, const double* w, const uint64_t* z, uint64_t start, int64_t count, double* out,
                   int device) {
  if (n < 2 || n > 63) return fail(LRQ_EVALIDATION, "num_qubits out of range [2, 63]");
  if (!w || !out || count < 0) return fail(LRQ_EVALIDATION, "null argument");
  if (count == 0) return LRQ_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRQ_ERUNTIME, "no CUDA device available (cut values have no CPU path)");
  DeviceGuard guard(device);
  const int E = n * (n - 1) / 2;
  double *dw = nullptr, *dout = nullptr;
  unsigned long long* dz = nullptr;
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t e = cudaMalloc(&dw, sizeof(double) * E);
  if (e == cudaSuccess) e = cudaMalloc(&dout, sizeof(double) * count);
  if (e == cudaSuccess && z) e = cudaMalloc(&dz, sizeof(unsigned long long) * count);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dw, w, sizeof(double) * E, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && z) e = cudaMemcpyAsync(dz, z, sizeof(uint64_t) * count, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    const long long blocks = (count + 255) / 256;
    cut_values_kernel<<<(unsigned)(blocks < 65535 ? blocks : 65535), 256, sizeof(double) * E, st>>>(
        n, dw, dz, count, (unsigned long long)start, dout);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, dout, sizeof(double) * count, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dw);
  cudaFree(dout);
  cudaFree(dz);
  cudaStreamDestroy(st);
  CUDA_TRY(e);
  return LRQ_OK;
}

}  // extern "C"

namespace {
// one-shot device scratch of the host-array entry points below: a stream and
// the buffers, freed on every path
struct Scratch {
  int device;
  cudaStream_t st = nullptr;
  std::vector<void*> bufs;
  explicit Scratch(int d) : device(d) {}
  cudaError_t init() { return cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); }
  template <typename P>
  cudaError_t alloc(P** p, size_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes ? bytes : 8);
    if (e == cudaSuccess) bufs.push_back(q);
    *p = reinterpret_cast<P*>(q);
    return e;
  }
  ~Scratch() {
    if (st) cudaStreamSynchronize(st);
    for (void* q : bufs) cudaFree(q);
    if (st) cudaStreamDestroy(st);
  }
};

int need_device(const char* what) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRQ_ERUNTIME, std::string("no CUDA device available (") + what + " has no CPU path)");
  return LRQ_OK;
}
}  // namespace

extern "C" {

int lrq_cut_values_spin(int n, const double* w, double half_total, uint64_t start, int64_t count, double* out,
                        int device) {
  if (n < 2 || n > 63) return fail(LRQ_EVALIDATION, "num_qubits out of range [2, 63]");
  if (!w || !out || count < 0) return fail(LRQ_EVALIDATION, "null argument");
  if (count == 0) return LRQ_OK;
  if (int rc = need_device("cut values")) return rc;
  DeviceGuard guard(device);
  std::vector<double> A((size_t)n * n);
  sym_matrix(n, w, A.data());
  Scratch sc(device);
  double *dA = nullptr, *dout = nullptr;
  cudaError_t e = sc.init();
  if (e == cudaSuccess) e = sc.alloc(&dA, sizeof(double) * n * n);
  const int64_t step = 1ll << 26;
  if (e == cudaSuccess) e = sc.alloc(&dout, sizeof(double) * (count < step ? count : step));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, sc.st);
  for (int64_t off = 0; e == cudaSuccess && off < count; off += step) {
    const int64_t m = count - off < step ? count - off : step;
    const long long blocks = (m + 255) / 256;
    cut_values_spin_kernel<<<(unsigned)(blocks < 65535 ? blocks : 65535), 256, sizeof(double) * n * n, sc.st>>>(
        n, dA, half_total, (unsigned long long)(start + off), m, dout);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out + off, dout, sizeof(double) * m, cudaMemcpyDeviceToHost, sc.st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(sc.st);
  }
  CUDA_TRY(e);
  return LRQ_OK;
}

int lrq_expected_cut(int n, const double* w, double half_total, const double* probs, uint64_t count,
                     double* chunk_sums, int device) {
  if (n < 2 || n > 40) return fail(LRQ_EVALIDATION, "num_qubits out of range [2, 40]");
  if (!w || !probs || !chunk_sums) return fail(LRQ_EVALIDATION, "null argument");
  if (count != (1ull << n)) return fail(LRQ_EVALIDATION, "distribution size must be 2^n");
  if (int rc = need_device("expected cut")) return rc;
  DeviceGuard guard(device);
  const int cb = n < 16 ? n : 16;  // reference chunk: 2^16 (engine.py:29)
  const long long chunks = (long long)(count >> cb);
  std::vector<double> A((size_t)n * n);
  sym_matrix(n, w, A.data());
  Scratch sc(device);
  double *dA = nullptr, *dp = nullptr, *ds = nullptr;
  cudaError_t e = sc.init();
  if (e == cudaSuccess) e = sc.alloc(&dA, sizeof(double) * n * n);
  if (e == cudaSuccess) e = sc.alloc(&dp, sizeof(double) * count);
  if (e == cudaSuccess) e = sc.alloc(&ds, sizeof(double) * chunks);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dA, A.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, sc.st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, probs, sizeof(double) * count, cudaMemcpyHostToDevice, sc.st);
  if (e == cudaSuccess) {
    expected_cut_kernel<<<(unsigned)chunks, 256, sizeof(double) * n * n, sc.st>>>(n, dA, half_total, dp,
                                                                                   (long long)count, cb, ds);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(chunk_sums, ds, sizeof(double) * chunks, cudaMemcpyDeviceToHost, sc.st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sc.st);
  CUDA_TRY(e);
  return LRQ_OK;
}

int lrq_draw_indices(const double* probs, uint64_t count, const double* u, int64_t shots, uint64_t* idx_out,
                     int device) {
  if (!probs || !u || !idx_out) return fail(LRQ_EVALIDATION, "null argument");
  if (shots < 1) return fail(LRQ_EVALIDATION, "shot count must be positive, got " + std::to_string(shots));
  if (count < 1) return fail(LRQ_EVALIDATION, "statevector has zero norm, nothing to sample");
  if (int rc = need_device("draw_indices")) return rc;
  DeviceGuard guard(device);
  int tb = 0;
  while (tb < 12 && (1ull << tb) < count) ++tb;
  const long long T = (long long)((count + (1ull << tb) - 1) >> tb);
  Scratch sc(device);
  double *dp = nullptr, *red = nullptr, *prefix = nullptr, *out = nullptr, *fin = nullptr, *du = nullptr;
  unsigned long long* didx = nullptr;
  cudaError_t e = sc.init();
  if (e == cudaSuccess) e = sc.alloc(&dp, sizeof(double) * count);
  if (e == cudaSuccess) e = sc.alloc(&red, sizeof(double) * kRedArrays * T);
  if (e == cudaSuccess) e = sc.alloc(&prefix, sizeof(double) * (T + 1));
  if (e == cudaSuccess) e = sc.alloc(&out, sizeof(double) * kOutScalars);
  if (e == cudaSuccess) e = sc.alloc(&fin, sizeof(double) * kFinScratch);
  if (e == cudaSuccess) e = sc.alloc(&du, sizeof(double) * shots);
  if (e == cudaSuccess) e = sc.alloc(&didx, sizeof(unsigned long long) * shots);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, probs, sizeof(double) * count, cudaMemcpyHostToDevice, sc.st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(du, u, sizeof(double) * shots, cudaMemcpyHostToDevice, sc.st);
  // the finalize reads all four partial arrays: zero sums, +inf minima
  if (e == cudaSuccess) e = cudaMemsetAsync(red + T, 0, sizeof(double) * T, sc.st);
  if (e == cudaSuccess) e = cudaMemsetAsync(red + 2 * T, 0x7f, sizeof(double) * T, sc.st);
  if (e == cudaSuccess) e = cudaMemsetAsync(red + 3 * T, 0xff, sizeof(double) * T, sc.st);
  if (e == cudaSuccess) {
    prob_tile_sums_kernel<<<(unsigned)((T * 32 + 255) / 256), 256, 0, sc.st>>>(dp, (long long)count, tb, T, red);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && launch_finalize(sc.st, T, red, prefix, out, fin) != LRQ_OK) e = cudaErrorUnknown;
  double total = 0.0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&total, out, sizeof(double), cudaMemcpyDeviceToHost, sc.st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(sc.st);
  CUDA_TRY(e);
  if (!(total > 0.0)) return fail(LRQ_EVALIDATION, "statevector has zero norm, nothing to sample");
  sample_probs_kernel<<<(unsigned)((shots * 32 + 255) / 256), 256, 0, sc.st>>>(dp, (long long)count, tb, T, prefix,
                                                                                du, shots, didx);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(idx_out, didx, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, sc.st));
  CUDA_TRY(cudaStreamSynchronize(sc.st));
  return LRQ_OK;
}

int lrq_max_cut(int n, const double* w, int device, uint64_t* argmax, double* value) {
  if (n < 2 || n > 48) return fail(LRQ_EVALIDATION, "num_qubits out of range [2, 48]");
  if (!w || !argmax || !value) return fail(LRQ_EVALIDATION, "null argument");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(LRQ_ERUNTIME, "no CUDA device available (max cut has no CPU path)");
  DeviceGuard guard(device);
  const int K = tile_amp_bits(8);
  uint64_t best = 0;
  if (n < K) {
    // tiny: reuse the whole-state kernel with p = 0 (uniform state) for min E
    lrq_state* s = nullptr;
    int rc = lrq_create(n, 16, device, 0, &s);
    if (rc) return rc;
    rc = lrq_set_cost(s, w);
    if (!rc) {
      SmallParams sp;
      memset(&sp, 0, sizeof sp);
      sp.amps = s->amps;
      sp.n = n;
      sp.p = 0;
      sp.J = s->dW;
      sp.mix = s->dzero;
      sp.W = s->dW;
      sp.init_re = 1.0;
      sp.min_bit = n - 1;
      double* rp = s->red;
      sp.red_p = rp;
      sp.red_pE = rp + 1;
      sp.red_minE = rp + 2;
      sp.red_arg = reinterpret_cast<unsigned long long*>(rp + 3);
      sp.red_maxE = rp + 4;
      rc = launch_small_any(16, sp, s->stream);
      cudaError_t e = rc ? cudaErrorUnknown : cudaSuccess;
      if (e == cudaSuccess) e = cudaMemcpyAsync(&best, rp + 3, 8, cudaMemcpyDeviceToHost, s->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
      if (e != cudaSuccess) rc = fail(LRQ_ERUNTIME, std::string("max cut: ") + cudaGetErrorString(e));
    }
    lrq_destroy(s);
    if (rc) return rc;
  } else {
    // exhaustive E_w scan over z with top bit 0 (complement symmetry), NOAMPS sweep
    const long long tiles = 1ll << (n - K - 1 >= 0 ? n - K - 1 : 0);
    const long long T = (n - 1 >= K) ? tiles : 1;
    double *dW = nullptr, *red = nullptr, *prefix = nullptr, *out = nullptr, *zero = nullptr, *fin = nullptr;
    cudaStream_t st;
    CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<double> M((size_t)n * n);
    sym_matrix(n, w, M.data());
    cudaError_t e = cudaMalloc(&dW, sizeof(double) * n * n);
    if (e == cudaSuccess) e = cudaMalloc(&red, sizeof(double) * kRedArrays * T);
    if (e == cudaSuccess) e = cudaMalloc(&prefix, sizeof(double) * (T + 1));
    if (e == cudaSuccess) e = cudaMalloc(&out, sizeof(double) * kOutScalars);
    if (e == cudaSuccess) e = cudaMalloc(&zero, sizeof(double) * (n + 1));
    if (e == cudaSuccess) e = cudaMalloc(&fin, sizeof(double) * kFinScratch);
    if (e == cudaSuccess) e = cudaMemsetAsync(zero, 0, sizeof(double) * (n + 1), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(red, 0, sizeof(double) * 2 * T, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dW, M.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      SweepParams sp;
      memset(&sp, 0, sizeof sp);
      sp.n = n;
      sp.q0 = K;
      sp.num_tiles = T;
      sp.reduce = 1;
      sp.scale_re = 1.0;
      sp.W.M = dW;
      sp.W.ext = zero;
      sp.J.M = dW;
      sp.J.ext = zero;
      sp.min_bit = n - 1;
      sp.red_p = red;
      sp.red_pE = red + T;
      sp.red_minE = red + 2 * T;
      sp.red_arg = reinterpret_cast<unsigned long long*>(red + 3 * T);
      sp.red_maxE = red + 4 * T;
      const int grid_cap = 2 * sm_count(device);
      const int grid = (int)(T < grid_cap ? T : grid_cap);
      const size_t smem = sweep_smem_bytes(n, false, false, true);
      if (launch_sweep_t<float, GK_A, SK_N>(st, sp, grid, smem) != LRQ_OK) e = cudaErrorUnknown;
    }
    if (e == cudaSuccess) {
      if (launch_finalize(st, T, red, prefix, out, fin) != LRQ_OK) e = cudaErrorUnknown;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&best, out + 3, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(dW);
    cudaFree(red);
    cudaFree(prefix);
    cudaFree(out);
    cudaFree(zero);
    cudaFree(fin);
    cudaStreamDestroy(st);
    CUDA_TRY(e);
  }
  *argmax = best;
  return lrq_cut_values(n, w, &best, 0, 1, value, device);
}

int lrq_set_search(lrq_state* s, int on) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  s->search = on != 0;
  return LRQ_OK;
}

int lrq_set_histogram(lrq_state* s, int bins, double lo, double hi) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  if (bins < 0 || bins > 4096) return fail(LRQ_EVALIDATION, "histogram bins must be in [0, 4096]");
  if (bins && !(isfinite(lo) && isfinite(hi) && hi > lo)) return fail(LRQ_EVALIDATION, "histogram range must be finite, hi > lo");
  DeviceGuard guard(s->device);
  if (bins != s->hist_bins) {
    cudaFree(s->dhist);
    s->dhist = nullptr;
    s->hist_bins = 0;
    if (bins) {
      CUDA_TRY(cudaMalloc(&s->dhist, sizeof(unsigned long long) * bins));
      CUDA_TRY(cudaMemsetAsync(s->dhist, 0, sizeof(unsigned long long) * bins, s->stream));
      CUDA_TRY(cudaStreamSynchronize(s->stream));
    }
  }
  s->hist_bins = bins;
  s->hist_lo = lo;
  s->hist_hi = hi;
  s->hist_valid = false;  // the next reducing pass fills it (the other reductions stay valid)
  return LRQ_OK;
}

int lrq_get_histogram(lrq_state* s, uint64_t* raw) {
  if (!s || !raw) return fail(LRQ_EVALIDATION, "null argument");
  if (!s->dhist) return fail(LRQ_ERUNTIME, "no histogram: call lrq_set_histogram, then run or recompute");
  if (!s->hist_valid) return fail(LRQ_ERUNTIME, "no histogram yet: run the circuit or recompute after lrq_set_histogram");
  DeviceGuard guard(s->device);
  const int B = s->hist_bins;
  if (s->world > 1 && !s->group) {
    if (!s->comm) return fail(LRQ_ERUNTIME, "aborted run: the communicator was aborted");
    // integer sums: the same result in any reduction order; afterwards every
    // rank holds the total (until the next reducing pass re-zeroes it)
    if (!s->hist_summed)
      NCCL_TRY_S(s, nccl().AllReduce(s->dhist, s->dhist, B, ncclUint64, ncclSum, s->comm, s->stream));
    CUDA_TRY(cudaMemcpyAsync(raw, s->dhist, sizeof(uint64_t) * B, cudaMemcpyDeviceToHost, s->stream));
    const int rc = dist_wait(s, s->stream);
    s->hist_summed = rc == LRQ_OK;
    return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(raw, s->dhist, sizeof(uint64_t) * B, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (s->group) {
    lrq_group* G = s->group;
    {
      std::lock_guard<std::mutex> lk(G->mu);
      G->shot_bufs[s->rank] = raw;
    }
    int rc = group_barrier(G);
    if (rc) return rc;
    std::vector<uint64_t> sum((size_t)B, 0);
    for (int r = 0; r < G->world; ++r)
      for (int b = 0; b < B; ++b) sum[b] += G->shot_bufs[r][b];
    rc = group_barrier(G);
    if (rc) return rc;
    memcpy(raw, sum.data(), sizeof(uint64_t) * B);
  }
  return LRQ_OK;
}

int lrq_set_timing(lrq_state* s, int enable) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  s->timing = enable != 0;
  return LRQ_OK;
}

int lrq_get_timings(lrq_state* s, double* ms, char* kinds, int cap, int* count) {
  if (!s || !count) return fail(LRQ_EVALIDATION, "null argument");
  const int c = (int)s->last_ms.size();
  *count = c;
  for (int i = 0; i < c && i < cap; ++i) {
    if (ms) ms[i] = s->last_ms[i];
    if (kinds) kinds[i] = i < (int)s->kinds.size() ? s->kinds[i] : '?';
  }
  return LRQ_OK;
}

int lrq_stream(lrq_state* s, void** out) {
  if (!s || !out) return fail(LRQ_EVALIDATION, "null argument");
  *out = (void*)s->stream;
  return LRQ_OK;
}

int lrq_synchronize(lrq_state* s) {
  if (!s) return fail(LRQ_EVALIDATION, "null state");
  DeviceGuard guard(s->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return LRQ_OK;
}

}  // extern "C"
