/* lrq.h — C ABI of the B200-native LR-QAOA state-vector engine (liblrq.so).
 *
 * Drop-in boundary for the reference package lrqbench (pure Python/numpy,
 * /root/reference/pkg/src/lrqbench).  Every entry point below replaces one
 * reference interface; the Python mirror paper_2604_26423_b200 binds them
 * with ctypes (see INTEGRATION.md for the binding a maintainer would add to
 * the reference itself).
 *
 * Conventions
 *   - plain C types only; host pointers unless a name says _dev;
 *   - basis index z has qubit/vertex k at bit k (engine.py:3-4);
 *   - edge arrays are in lexicographic (i<j) order, length n(n-1)/2
 *     (problem.py:32-34);
 *   - return codes mirror the reference exception taxonomy / CLI exit codes
 *     (errors.py:8-26, cli.py:64-67): 0 ok, 2 ValidationError,
 *     3 CapacityError, 4 StateError/AbortedRunError (runtime);
 *     lrq_last_error() gives the message of the calling thread's last failure.
 */
#ifndef LRQ_H
#define LRQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRQ_OK 0
#define LRQ_EVALIDATION 2
#define LRQ_ECAPACITY 3
#define LRQ_ERUNTIME 4

#define LRQ_ABI_VERSION 2

typedef struct lrq_state lrq_state; /* one state vector (or one rank's shard) in HBM */

typedef struct lrq_reduction {
  double sum_p;        /* sum_z |a_z|^2 (float64)                          */
  double sum_p_cut;    /* sum_z |a_z|^2 C(z)  -> exact r = sum_p_cut / C*  */
  double min_energy;   /* min_z E_w(z) over z with top bit 0 (spin form)   */
  uint64_t argmax_cut; /* lowest-index z attaining it (= argmax C)         */
  double max_energy;   /* max_z E_w(z) (= W - 2 min C: the minimum cut)     */
} lrq_reduction;

/* library / device ------------------------------------------------------- */
int lrq_abi_version(void);
const char *lrq_last_error(void);
int lrq_device_count(int *count);

/* Host-only: JSON description of the sweep plan for (n, precision_bytes, p).
 * No GPU needed; used by CPU tests of the planner.                          */
int lrq_describe_plan(int num_qubits, int precision_bytes, int p, char *buf, size_t cap);

/* state lifecycle — replaces engine.py:99-110 zero_state/check_memory.
 * precision_bytes: 8 = complex64 (Precision.FP32), 16 = complex128 (FP64).
 * memory_budget: bytes allowed for the state; 0 = device capacity.
 * Over budget -> 3 with the reference's message shape (engine.py:67-74).   */
int lrq_create(int num_qubits, int precision_bytes, int device, uint64_t memory_budget, lrq_state **out);
int lrq_destroy(lrq_state *s);

/* cost function for the fused final pass: edge weights w (lex order),
 * replaces the WmcInstance consumed by exact_expected_r (engine.py:229-235). */
int lrq_set_cost(lrq_state *s, const double *w);

/* run_circuit (engine.py:198-207) for an H-layer + p x (RZZ*, RX^n) circuit:
 *   phase[k*E + e] = sum of theta/2 over the layer-k RZZ gates on edge e,
 *   mixer[k]       = theta/2 of the layer-k RX gates (same on every qubit).
 * Starts from |0..0>, applies the H layer, the p layers, and (if a cost was
 * set) the fused final pass.  Synchronous.                                  */
int lrq_run(lrq_state *s, int p, const double *phase, const double *mixer);

/* lrq_run with, per layer k, extra diagonal terms in the cost phase:
 *   exp(-i (sum_e phase[k*E+e] Z_i Z_j + sum_i field[k*n+i] Z_i + constant[k])).
 * Single-GPU.  The reference circuits (H, RZZ, RX; circuit.py:66-81) never
 * need it; it is the single-device form of the rank-local terms the
 * multi-GPU engine derives from the global qubits (lrq_dist_terms).        */
int lrq_run_fields(lrq_state *s, int p, const double *phase, const double *field, const double *constant,
                   const double *mixer);

/* lrq_run with per-qubit mixer half-angles mixer_q[k*n + q] that agree up to
 * sign within each layer (noisy trajectories: Z/Y Paulis flip RX angles), and
 * the X string left at the end of a trajectory: z <-> z ^ mask.  Single GPU. */
int lrq_run_ex(lrq_state *s, int p, const double *phase, const double *mixer_q);
int lrq_permute_xor(lrq_state *s, uint64_t mask);

/* Gate-by-gate execution (engine.py:99-195) for circuits of any other shape:
 * reset to |0...0> (which = 0) or to the uniform state 2^(-n/2) (which = 1,
 * init_plus_state), then apply H (kind 0), RX(theta) (1) or RZZ(theta) (2)
 * one full pass at a time, with the reference kernels' complex arithmetic,
 * or a Pauli X (3), Y (4), Z (5) on q0 (exact; the noisy engine's Pauli
 * insertions, noise.py:70-98).
 * Asynchronous on the engine stream; lrq_recompute / lrq_sample after.     */
int lrq_reset(lrq_state *s, int which);
int lrq_apply_gate(lrq_state *s, int kind, int q0, int q1, double theta);

/* Noisy Monte Carlo trajectories (noise.py:109-207) for small n (n below the
 * tile: 12 complex128 / 13 complex64), batched one trajectory per CTA.
 * Trajectory t is the ideal circuit with its Pauli insertions propagated to
 * the end: per-layer edge angles phase[(t*p + k)*E + e] (signs flipped by X/Y
 * insertions), per-qubit mixer half-angles mixer[(t*p + k)*n + q] (equal up
 * to sign within a layer; Z/Y flip the sign), and a final X mask xmask[t]
 * (probabilities permuted z -> z ^ mask).  Writes trajectory probabilities
 * (float64, T x 2^n, may be NULL) and, if shots > 0, inverse-CDF draws with
 * the caller's uniforms u[t*shots + i] into idx_out[t*shots + i].          */
int lrq_noisy_batch(int num_qubits, int precision_bytes, int device, int trajectories, int p, const double *phase,
                    const double *mixer, const unsigned *xmask, int64_t shots, const double *u, double *probs_out,
                    uint64_t *idx_out);

/* Whether the fused final pass (and lrq_recompute) also searches min E with
 * its lowest-index argmin (the exhaustive max cut, problem.py:174-211) and
 * max E.  On by default; a caller that already knows C* turns it off and the
 * pass only sums p and p*E (min_energy / max_energy / argmax_cut then read
 * +inf / -inf / ~0).                                                       */
int lrq_set_search(lrq_state *s, int on);

/* reductions of the last run (exact_expected_r numerator, engine.py:214-226;
 * exhaustive max cut argmax, problem.py:174-211).                            */
int lrq_reduce(lrq_state *s, lrq_reduction *out);

/* read-only pass: recompute the reductions and the sampler CDF from the
 * current state with the current cost (zero cost if none was set).         */
int lrq_recompute(lrq_state *s);

/* p-weighted histogram of the cost energy E_w(z) over `bins` equal bins of
 * [lo, hi) (values outside clamp to the end bins), filled by the fused final
 * pass of the next lrq_run / lrq_recompute (bins = 0: off, the default; on,
 * the reducing pass adds one shared-memory integer atomic per amplitude).
 * raw[b] = sum over z in bin b of round(|a_z|^2 2^60): integer sums, so the
 * result is identical in any order and on any number of ranks (collective:
 * summed over ranks).  Exact distribution of C = (W - E)/2 for the
 * chi-square test of sampled shots.                          */
int lrq_set_histogram(lrq_state *s, int bins, double lo, double hi);
int lrq_get_histogram(lrq_state *s, uint64_t *raw);

/* inverse-CDF sampling (engine.py:254-273) with caller-supplied uniforms
 * (the reference draws them from Philox("shots", 0) on the host).           */
int lrq_sample(lrq_state *s, const double *u, int64_t shots, uint64_t *idx_out);

/* amplitudes [start, start+count) -> host, complex64/complex128 interleaved;
 * lrq_store_amps: host -> state (LQSV load, engine.py:296-312).           */
int lrq_copy_amps(lrq_state *s, uint64_t start, uint64_t count, void *host_out);
int lrq_store_amps(lrq_state *s, uint64_t start, uint64_t count, const void *host_in);

/* bit-exact cut values (problem.py:139-149) on the device. z==NULL means the
 * contiguous range [start, start+count).                                    */
int lrq_cut_values(int num_qubits, const double *w, const uint64_t *z, uint64_t start, int64_t count,
                   double *out, int device);

/* spin-form cut values C = W/2 - s^T A s / 4 of the contiguous range
 * [start, start+count) — cut_values_range (problem.py:158-171); half_total =
 * 0.5 * WmcInstance.total_weight().  Equal to lrq_cut_values to ~1e-15.     */
int lrq_cut_values_spin(int num_qubits, const double *w, double half_total, uint64_t start, int64_t count,
                        double *out, int device);

/* numerator of expected_r_from_probs (engine.py:214-226) for an explicit
 * float64 distribution of 2^n entries: chunk_sums[c] = sum over the c-th 2^16
 * block of p_z * C_spin(z) (2^n / 2^16 outputs, or 1 for n < 16); the caller
 * adds them in order.                                                       */
int lrq_expected_cut(int num_qubits, const double *w, double half_total, const double *probs, uint64_t count,
                     double *chunk_sums, int device);

/* draw_indices (engine.py:254-263) over an explicit float64 distribution:
 * first index whose normalised cumulative probability exceeds u[i], clamped
 * to count-1.  Zero total mass -> 2 ("statevector has zero norm").         */
int lrq_draw_indices(const double *probs, uint64_t count, const double *u, int64_t shots, uint64_t *idx_out,
                     int device);

/* exhaustive max cut (optimal_cut_bruteforce, problem.py:174-211) on the
 * device: lowest-index argmax of C; value re-evaluated bit-exactly.         */
int lrq_max_cut(int num_qubits, const double *w, int device, uint64_t *argmax, double *value);

/* multi-GPU (one process per GPU) — replaces the shard threads of
 * run_circuit_sharded (sharded.py:202-385).  world = 2^g ranks; rank r holds
 * the 2^(n-g) amplitudes whose top g bits equal r.  All ranks call lrq_run,
 * lrq_reduce and lrq_sample collectively (NCCL inside); lrq_sample returns
 * the same global indices on every rank; lrq_copy_amps reads the local shard.
 * nccl_id: 128 bytes from lrq_nccl_unique_id on one rank, shared by the host. */
int lrq_nccl_unique_id(void *out, size_t cap);
int lrq_create_dist(int num_qubits, int precision_bytes, int device, int rank, int world, const void *nccl_id,
                    uint64_t memory_budget, lrq_state **out);
int lrq_dist_info(lrq_state *s, int *n_local, int *rank, int *world);

/* An odd number of layers leaves a distributed state with its g global
 * qubits and top g local qubits swapped (the run makes one remap per layer
 * and no restoring one).  Reductions and sampling work in either layout;
 * reading or writing the shard's amplitudes needs the identity layout:
 * lrq_restore_layout (collective) makes the remaining remap and recomputes
 * the reductions; lrq_copy_amps refuses a swapped shard.  layout_out of
 * lrq_dist_layout: 0 identity, 1 swapped.                                 */
int lrq_restore_layout(lrq_state *s);
int lrq_dist_layout(lrq_state *s, int *layout_out);

/* Remap transports over peer memory (NVLink).  Collective setup: every rank
 * exports its buffers (lrq_ipc_handles, LRQ_IPC_HANDLE_BYTES bytes), the host
 * gathers them in rank order (world * LRQ_IPC_HANDLE_BYTES bytes) and every
 * rank calls lrq_fused_setup, which maps the peers' buffers and runs a
 * peer-store self-test.  *enabled (the same on all ranks):
 *   1  fused remap: every rank holds a spare state buffer, and the sweep
 *      before a remap stores every block straight into its owner's spare;
 *   2  pipelined remap over peer memory: the sweep before a remap runs block
 *      by block and each finished block is swapped in place with its owner
 *      (XOR schedule, no second buffer: the case at the HBM limit);
 *   0  NCCL send/recv remap (pipelined the same way, through a staging chunk).
 * The spare buffer is taken only if it fits with 2 GiB to spare.  In-process
 * shard groups use the members' buffers directly.  LRQ_FUSED_REMAP=0 disables
 * the fused form, LRQ_PIPELINED_REMAP=0 the block pipelining.            */
#define LRQ_IPC_HANDLE_BYTES 256
int lrq_ipc_handles(lrq_state *s, void *out, size_t cap);
int lrq_fused_setup(lrq_state *s, const void *all_handles, int *enabled);

/* Host-only accounting: device bytes one rank allocates for an n-qubit state
 * over `world` ranks (world 1: the single-GPU engine) at depth p — the state,
 * reductions, cost matrices and (NCCL transport) the staging chunk; the
 * fused remap's optional spare buffer is extra_spare.                      */
/* Host-only: the remap schedule of `rank` as JSON [[partner, my_block,
 * their_block, half], ...] — the XOR pairwise steps of the all-to-all block
 * transpose (mirror < 0) or the one whole-state step with rank `mirror`
 * (block -1) of the deferred global flip.                                  */
int lrq_describe_remap(int world, int rank, int mirror, char *buf, size_t cap);

int lrq_describe_memory(int num_qubits, int precision_bytes, int world, int p, uint64_t *state_bytes,
                        uint64_t *other_bytes, uint64_t *extra_spare);

/* in-process shards — the B200 form of the reference's thread-per-shard
 * engine (run_circuit_sharded / _ShardWorker, sharded.py:200-385): `world`
 * shard states in ONE process, one host thread per shard making the same
 * collective calls as above (lrq_run, lrq_reduce, lrq_sample).  The shards
 * may share a device or sit on several (peer access).  The group replaces
 * NCCL with a host barrier and device-side block swaps; a failure in any
 * collective call aborts the whole group (AbortedRunError, errors.py:24-26).
 * Destroy the shard states before the group.                               */
typedef struct lrq_group lrq_group;
int lrq_group_create(int world, lrq_group **out);
int lrq_group_destroy(lrq_group *g);
int lrq_group_abort(lrq_group *g); /* break the group: blocked members return 4 */
int lrq_create_shard(int num_qubits, int precision_bytes, int device, int rank, lrq_group *g,
                     uint64_t memory_budget, lrq_state **out);

/* Host-only helpers of the distributed plan (CPU-testable): the JSON sweep /
 * remap schedule, and a rank's local view of a Z-Z coupling (lexicographic
 * edges) in permutation state perm: local matrix, field, constant.          */
int lrq_describe_dist_plan(int num_qubits, int log2_world, int precision_bytes, int p, char *buf, size_t cap);
int lrq_dist_terms(int num_qubits, int log2_world, int rank, int perm, const double *edges, double *local_matrix,
                   double *field, double *constant);

/* timing: per-launch device milliseconds of the last lrq_run (CUDA events on
 * the engine stream), plus the engine stream handle for external events.   */
int lrq_set_timing(lrq_state *s, int enable);
int lrq_get_timings(lrq_state *s, double *ms, char *kinds, int cap, int *count);
int lrq_stream(lrq_state *s, void **stream_out);
int lrq_synchronize(lrq_state *s);

#ifdef __cplusplus
}
#endif
#endif /* LRQ_H */
