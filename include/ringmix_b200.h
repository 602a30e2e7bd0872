/*
 * ringmix_b200 — C-ABI of the B200-native learner-averaging hot path.
 *
 * The reference (arXiv 2002.01119 simulator `ringmix`, pure Python/numpy) has
 * no FFI; its plugin surface for this path is a set of Python functions.  Each
 * entry point below replaces one of them (file:line under /root/reference):
 *
 *   rm_perm_tables        <- mixing.permutation_for_step     pkg/src/ringmix/mixing.py:79-86
 *                            (+ the conjugation T0[p, p] of  simulation.py:299-300 /
 *                             mixing.conjugate_by_permutation mixing.py:89-103,
 *                             reduced to neighbour tables)
 *   rm_perm_sequential    <- seeding.stream + repeated        seeding.py:35-37,
 *                            mixing.sample_permutation        mixing.py:72-76
 *                            as drawn by monte_carlo_consensus spectral.py:273-277
 *   rm_pcg64_raw          <- numpy PCG64.random_raw under SeedSequence (pins the core)
 *   rm_ring_mix_sgd_*     <- simulation._gossip_step          simulation.py:263-268
 *                            = apply_mixing(W, T) - lr*G      mixing.py:106-125
 *                            for T = ring or ring[p, p]       (step_rand_psgd :285-301,
 *                                                              step_dpsgd_fixed :271-273,
 *                                                              step_adpsgd_fixed :276-282)
 *                            with the fused _check_divergence  simulation.py:390-395
 *   rm_mean_sgd_*         <- step_d1d / uniform apply_mixing   simulation.py:304-312,
 *                                                              mixing.py:122-124
 *   rm_spsgd_*            <- step_spsgd                        simulation.py:251-260
 *   rm_*_host_f32         <- the same step on HOST buffers (H2D, kernel, D2H pipelined)
 *   rm_gossip_step_dL_* / rm_gossip_step_host_dL_*
 *                         <- the same step on the reference's own (d, L) C-order arrays
 *                            (device or host), ring or uniform T   simulation.py:263-268
 *   rm_quadratic_grad_*   <- simulation.gradient_matrix with   simulation.py:226-238,
 *   (and _shard_*)           QuadraticObjective.stochastic_   objectives.py:84-90
 *                            gradient (bit-exact numpy normals)
 *   rm_quadratic_mix_step_* <- gradient_matrix + _gossip_step  simulation.py:226-238 +
 *                            in one pass (G never in HBM)      :263-268 / :304-312
 *   rm_standard_normal_f64 <- seeding.stream(...).standard_normal  seeding.py:35-37
 *   rm_trace_stats_*      <- run_training._record: consensus   simulation.py:398-409,
 *                            distance + loss_columns + loss   :359-362, objectives.py:77-79
 *   rm_column_mean_*      <- W.mean(axis=1) of step_d1d        mixing.py:122-124
 *   rm_ring_mix_batched_f64 <- product @ T_k of                spectral.py:273-279
 *                            monte_carlo_consensus
 *   rm_ipc_* / rm_shard_* / rm_pos_* / rm_partial_sum_* / rm_apply_mean_sgd_* /
 *   rm_nvls_mean_f64 / rm_p2p_mean_f64 / rm_d1d_fused_* / rm_step_sync_wait /
 *   rm_xgpu_status
 *                         <- (no reference counterpart: the reference simulates all
 *                            learners in one process; these shard them over GPUs —
 *                            the step they compute is still simulation.py:263-268 /
 *                            :304-312)
 *
 * Conventions
 *   - All compute pointers are caller-owned DEVICE memory unless the name says
 *     `host`; nothing here allocates device memory.
 *   - Weights are learner-major: row l (learner l) starts at base + l*ld
 *     elements.  The reference's (d, L) matrix is the transpose view.
 *   - Calls are stream-ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *   - Return 0 on success; a negative RM_E* code for bad arguments; a positive
 *     cudaError_t for CUDA failures.  rm_last_error() gives a thread-local
 *     message (the reference's ValueError text where one exists).
 *   - Safe to call from several host threads on distinct streams.
 *   - W and Wout must not alias (cross-learner read-after-write hazard).
 *   - absmax_bits (optional): receives atomicMax of the IEEE-754 bit pattern of
 *     |W'| as a double; > 0x7ff0000000000000 means NaN, == means inf.  Caller
 *     zeroes it.
 */
#ifndef RINGMIX_B200_H
#define RINGMIX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RM_EINVAL (-1)
#define RM_ENOSYS (-2)
#define RM_ERANGE (-3)
#define RM_ETIMEDOUT (-4)

const char* rm_last_error(void);
int rm_version(void);
int rm_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);
/* For FFI callers without a CUDA runtime of their own (the reference's numpy code through
 * ctypes): a device buffer (e.g. the host-step workspace), a stream-ordered copy in any
 * direction (cudaMemcpyDefault), and a stream synchronise. */
int rm_device_alloc(int64_t bytes, void** ptr);
int rm_device_free(void* ptr);
int rm_memcpy(void* dst, const void* src, int64_t bytes, void* stream);
int rm_stream_synchronize(void* stream);
/* Single-process multi-GPU: enable peer access between every pair of devices 0..ndev-1
 * (already-enabled pairs are fine; RM_ENOSYS if a pair has no P2P path). */
int rm_enable_peer_access(int ndev);

/* ---- permutations (bit-exact with numpy 2.3.5 SeedSequence/PCG64/permutation) ----
 * prefix_words: the entropy words of (seed, tag) — numpy's
 * _coerce_to_uint32_array: each int as little-endian u32 limbs, 0 -> [0] —
 * computed by the caller (any size of seed).  The kernel appends limbs(step).
 * perm/inv (required) and left/right (optional) are int32[nsteps][L]. */
int rm_perm_tables(const uint32_t* prefix_words, int n_prefix, uint64_t step0, int nsteps, int L,
                   int32_t* perm, int32_t* inv, int32_t* left, int32_t* right, void* stream);

/* nstreams independent streams (entropy prefix + limbs(idx0 + s)); each draws
 * `count` permutations back to back.  perms: int32[nstreams][count][L]. */
int rm_perm_sequential(const uint32_t* prefix_words, int n_prefix, uint64_t idx0, int nstreams,
                       int count, int L, int32_t* perms, void* stream);

/* Stateful streams (the Generator objects seeding.stream returns).  A state is
 * 6 x uint64 in device memory.  rm_pcg_seed seeds nstreams states from
 * prefix (+ limbs(idx0 + s) when with_index); rm_pcg_permutations draws
 * `count` permutations per state back to back and writes the advanced state
 * back, so successive calls continue the stream exactly like repeated
 * Generator.permutation calls. */
int rm_pcg_seed(const uint32_t* prefix_words, int n_prefix, int with_index, uint64_t idx0,
                int nstreams, uint64_t* states, void* stream);
int rm_pcg_permutations(uint64_t* states, int nstreams, int count, int L, int32_t* perms,
                        void* stream);

/* count raw next64() outputs of PCG64(SeedSequence(entropy_words)). */
int rm_pcg64_raw(const uint32_t* entropy_words, int n_words, int count, uint64_t* out,
                 void* stream);

/* ---- fused mix + SGD:  Wout[j] = (W[left j] + W[j] + W[right j])/3 - lr*G[j] ----
 * G may be NULL (pure apply_mixing).  L == 3 takes the exact column-mean path
 * like the reference (mixing.py:122-124).  fp32/fp64 compute in fp64 with the
 * reference's rounding sequence; bf16 (uint16_t storage) computes in fp32. */
int rm_ring_mix_sgd_f32(const float* W, const float* G, float* Wout, const int32_t* left,
                        const int32_t* right, int L, int64_t d, int64_t ldw, int64_t ldg,
                        int64_t ldo, double lr, unsigned long long* absmax_bits, void* stream);
int rm_ring_mix_sgd_f64(const double* W, const double* G, double* Wout, const int32_t* left,
                        const int32_t* right, int L, int64_t d, int64_t ldw, int64_t ldg,
                        int64_t ldo, double lr, unsigned long long* absmax_bits, void* stream);
int rm_ring_mix_sgd_bf16(const uint16_t* W, const uint16_t* G, uint16_t* Wout,
                         const int32_t* left, const int32_t* right, int L, int64_t d, int64_t ldw,
                         int64_t ldg, int64_t ldo, double lr, unsigned long long* absmax_bits,
                         void* stream);

/* ---- D1D / uniform:  Wout[j] = mean_l W[l] - lr*G[j]  (numpy pairwise mean) ---- */
int rm_mean_sgd_f32(const float* W, const float* G, float* Wout, int L, int64_t d, int64_t ldw,
                    int64_t ldg, int64_t ldo, double lr, unsigned long long* absmax_bits,
                    void* stream);
int rm_mean_sgd_f64(const double* W, const double* G, double* Wout, int L, int64_t d,
                    int64_t ldw, int64_t ldg, int64_t ldo, double lr,
                    unsigned long long* absmax_bits, void* stream);
int rm_mean_sgd_bf16(const uint16_t* W, const uint16_t* G, uint16_t* Wout, int L, int64_t d,
                     int64_t ldw, int64_t ldg, int64_t ldo, double lr,
                     unsigned long long* absmax_bits, void* stream);

/* ---- S-PSGD:  Wout[j] = W[j] - lr*mean_l G[l];  *mismatch |= any(W[j] != W[0]) ---- */
int rm_spsgd_f32(const float* W, const float* G, float* Wout, int L, int64_t d, int64_t ldw,
                 int64_t ldg, int64_t ldo, double lr, unsigned int* mismatch,
                 unsigned long long* absmax_bits, void* stream);
int rm_spsgd_f64(const double* W, const double* G, double* Wout, int L, int64_t d, int64_t ldw,
                 int64_t ldg, int64_t ldo, double lr, unsigned int* mismatch,
                 unsigned long long* absmax_bits, void* stream);
int rm_spsgd_bf16(const uint16_t* W, const uint16_t* G, uint16_t* Wout, int L, int64_t d,
                  int64_t ldw, int64_t ldg, int64_t ldo, double lr, unsigned int* mismatch,
                  unsigned long long* absmax_bits, void* stream);

/* ---- host-buffer step (reference calling convention: arrays in host RAM) ----
 * W_host/G_host/out_host: (L, d) row-major fp32 in host memory (pinned for
 * overlap); left/right: host int32[L].  The step is pipelined over column
 * chunks (H2D || kernel || D2H) through `workspace` (device, workspace_bytes;
 * rm_host_chunk_cols reports the chunk width it allows).  Stream-ordered on
 * `stream`; the host buffers must stay valid until it completes.  Every calling host
 * thread has its own internal copy streams per device; concurrent calls need distinct
 * workspaces.  G_host may be NULL. */
int rm_host_chunk_cols(int L, int64_t workspace_bytes, int64_t* chunk_cols);
int rm_ring_mix_sgd_host_f32(const float* W_host, const float* G_host, float* out_host,
                             const int32_t* left_host, const int32_t* right_host, int L, int64_t d,
                             double lr, void* workspace, int64_t workspace_bytes,
                             unsigned long long* absmax_bits, void* stream);

/* ---- the reference's own array layout: (d, L) C-order ----
 * simulation._gossip_step / apply_mixing on the arrays the reference holds
 * (simulation.py:209, 263-268; mixing.py:106-125): W, G, W' are (d, L) row-major with
 * row strides ldw / ldg / ldo >= L (elements); row r is coordinate r of every learner.
 * left == right == NULL selects the uniform mean (D1D, mixing.py:122-124); otherwise
 * the ring / ring[p, p] gather with neighbour tables as rm_ring_mix_sgd_*.  Same
 * arithmetic and rounding as the learner-major kernels (no transpose anywhere). */
int rm_gossip_step_dL_f32(const float* W, const float* G, float* out, const int32_t* left,
                          const int32_t* right, int L, int64_t d, int64_t ldw, int64_t ldg,
                          int64_t ldo, double lr, unsigned long long* absmax_bits, void* stream);
int rm_gossip_step_dL_f64(const double* W, const double* G, double* out, const int32_t* left,
                          const int32_t* right, int L, int64_t d, int64_t ldw, int64_t ldg,
                          int64_t ldo, double lr, unsigned long long* absmax_bits, void* stream);
/* The same on HOST (d, L) C-order arrays (dense rows, ld = L), e.g. the reference's
 * numpy weights: contiguous row chunks H2D || kernel || D2H through `workspace` (device,
 * >= 4096 + 9 * rows * L * sizeof(T) bytes for a chunk of `rows` rows); left/right are
 * host int32[L] (or NULL for the uniform mean).  L <= 512.  Stream-ordered on `stream`;
 * the host arrays must stay valid until it completes. */
int rm_gossip_step_host_dL_f32(const float* W_host, const float* G_host, float* out_host,
                               const int32_t* left_host, const int32_t* right_host, int L,
                               int64_t d, double lr, void* workspace, int64_t workspace_bytes,
                               unsigned long long* absmax_bits, void* stream);
int rm_gossip_step_host_dL_f64(const double* W_host, const double* G_host, double* out_host,
                               const int32_t* left_host, const int32_t* right_host, int L,
                               int64_t d, double lr, void* workspace, int64_t workspace_bytes,
                               unsigned long long* absmax_bits, void* stream);

/* ---- learner-sharded multi-GPU path (one process per GPU) ----
 * CUDA IPC: export / map a peer process's device allocation (handles are
 * rm_ipc_handle_size() bytes, exchanged by the caller, e.g. torch.distributed).
 * offset_out = byte offset of dptr inside the exported allocation; the importer
 * adds it to the base rm_ipc_open_handle returns. */
int rm_ipc_handle_size(void);
int rm_ipc_get_handle(const void* dptr, void* handle_out, uint64_t* offset_out);
int rm_ipc_open_handle(const void* handle, void** dptr_out);
int rm_ipc_close_handle(void* dptr);

/* Optional in-kernel step ordering for the learner-sharded step kernels, replacing a
 * host-issued barrier between steps: the kernel of step `epoch` (1, 2, ...) waits until
 * *done >= world * (epoch - 1) — every rank finished the previous step, whose rows it reads
 * and whose buffers it overwrites — and at its end adds 1 to `done` on every rank through
 * the multicast address done_mc (multimem.red.release).  done: symmetric uint32, zeroed on
 * every rank before the first step; counter: local device uint32, zeroed once.
 * Without NVSwitch multicast (done_mc == NULL) done_peers, a device uint64[world] table of
 * every rank's `done` address (CUDA IPC / symmetric-memory peer pointers), is used instead:
 * one red.release per rank.  With every rank's buffers on one GPU the same table drives a
 * single-device emulation of the world (launch the ranks' steps in rank order per epoch).
 * A wait longer than RINGMIX_XGPU_TIMEOUT_S (default 600 s) gives up instead of trapping
 * and is reported by rm_xgpu_status(). */
typedef struct {
  const uint32_t* done;
  uint32_t* done_mc;
  uint32_t* counter;
  uint32_t epoch;
  int world;
  const uint64_t* done_peers;
} rm_step_sync;

/* Reads and clears the calling device's cross-rank wait status: bit 0 set = a cross-rank
 * wait (step ordering, fused D1D) gave up after RINGMIX_XGPU_TIMEOUT_S; the step that
 * saw it has unspecified contents. */
int rm_xgpu_status(unsigned int* status);
/* Sets the cross-rank wait bound of the current device (seconds; overrides the
 * RINGMIX_XGPU_TIMEOUT_S default). */
int rm_set_xgpu_timeout(double seconds);

/* Stream-ordered wait until every rank finished step `sync->epoch` (*done >= world *
 * epoch).  The next step kernel orders itself; any other consumer of a step's outputs
 * in the ring-position layout (whose rows are written by every rank) calls this first.
 * Returns 0 without launching when epoch == 0. */
int rm_step_sync_wait(const rm_step_sync* sync, void* stream);

/* Stream-ordered publish of writes made outside the step kernels (initial weights,
 * checkpoint restore, host edits of the current rows): adds 1 to `done` on every rank as a
 * step's end would.  Collective: every rank calls it once, with sync->epoch = the epoch it
 * occupies (last step + 1); the next step (epoch + 1) of every rank then waits for every
 * rank's writes.  Readers of the position layout's slots call rm_step_sync_wait first;
 * writers call rm_step_sync_wait (position layout: peers write into this rank's slots),
 * write, then rm_step_sync_publish. */
int rm_step_sync_publish(const rm_step_sync* sync, void* stream);

/* Per-step plan for the rank owning learners [row0, row0+Lg): distinct remote
 * neighbour ids and each local learner's staged input indices in global-id
 * order.  plan: device int32[rm_shard_plan_ints(Lg)]; left/right: device
 * int32[L] (the step's global tables from rm_perm_tables). */
int rm_shard_plan_ints(int Lg);
int rm_shard_plan(const int32_t* left, const int32_t* right, int L, int row0, int Lg,
                  int32_t* plan, void* stream);

/* Fused step for the local learners: out[j] = ring3(...) - lr*G_local[j]; local
 * rows by TMA, remote neighbour rows pulled from peer HBM over NVLink inside the
 * kernel.  row_ptrs: device uint64[L], row l of the current W of every rank
 * (local or IPC-mapped peer address).  Bit-identical to the single-GPU step.
 * The caller orders steps across ranks (a barrier between steps). */
int rm_ring_mix_sgd_sharded_f32(const uint64_t* row_ptrs, const float* W_local,
                                const float* G_local, float* out, int L, int row0, int Lg,
                                int64_t d, int64_t ldw, int64_t ldg, int64_t ldo,
                                const int32_t* plan, double lr, unsigned long long* absmax_bits,
                                void* stream,
                                const rm_step_sync* sync);
int rm_ring_mix_sgd_sharded_f64(const uint64_t* row_ptrs, const double* W_local,
                                const double* G_local, double* out, int L, int row0, int Lg,
                                int64_t d, int64_t ldw, int64_t ldg, int64_t ldo,
                                const int32_t* plan, double lr, unsigned long long* absmax_bits,
                                void* stream,
                                const rm_step_sync* sync);
int rm_ring_mix_sgd_sharded_bf16(const uint64_t* row_ptrs, const uint16_t* W_local,
                                 const uint16_t* G_local, uint16_t* out, int L, int row0, int Lg,
                                 int64_t d, int64_t ldw, int64_t ldg, int64_t ldo,
                                 const int32_t* plan, double lr,
                                 unsigned long long* absmax_bits, void* stream,
                                const rm_step_sync* sync);

/* RAD in ring-position order ("push" layout): the rank owning positions [g0, g0+Lg)
 * stores, in slot x, the learner at position x of step k (inv_k[x]).  rm_pos_plan
 * builds the step's plan (boundary positions g0-1 and g0+Lg are the only remote
 * reads) and dest[i] = address of learner inv_k[g0+i]'s slot for step k+1
 * (next_slot_ptrs[perm_next[learner]], any rank).  rm_ring_mix_sgd_pos_* then mixes
 * in position space (FMA chain in learner-id order: bit-identical to the
 * single-GPU step) and writes every output straight to its next-step slot. */
int rm_pos_plan(const int32_t* inv_k, const int32_t* perm_next, int L, int g0, int Lg,
                const uint64_t* next_slot_ptrs, int32_t* plan, uint64_t* dest, void* stream);
/* Placed ring-position layout: global slot s (rank s / Lg, row s % Lg) holds ring position
 * pos_of_slot[s] and position q lives in slot slot_of_pos[q] (device int32[L] each; every
 * rank's slots hold a contiguous arc of positions), slot_of_pos_next is step k+1's
 * placement.  rm_pos_plan is the identity placement (slot x = position x). */
int rm_pos_plan_placed(const int32_t* inv_k, const int32_t* perm_next, const int32_t* pos_of_slot,
                       const int32_t* slot_of_pos, const int32_t* slot_of_pos_next, int L, int g0,
                       int Lg, const uint64_t* next_slot_ptrs, int32_t* plan, uint64_t* dest,
                       void* stream);
/* Placement of step k+1 (L % world == 0, world <= 8, L <= 1024): the rotation of the arcs
 * and the arc -> rank assignment that keep the most learners on the rank computing their
 * output (fewest relabelling stores over NVLink), given step k's placement slot_of_pos
 * (NULL = identity), inv_k and perm_next.  Deterministic: every rank computes the same.
 * moved (optional, device int32[world]): learners leaving each rank in this relabelling. */
int rm_pos_placement(const int32_t* inv_k, const int32_t* perm_next, const int32_t* slot_of_pos,
                     int L, int world, int32_t* pos_of_slot_next, int32_t* slot_of_pos_next,
                     int32_t* moved, void* stream);
int rm_ring_mix_sgd_pos_f32(const uint64_t* slot_ptrs, const float* W_local, const float* G_local,
                            int L, int g0, int Lg, int64_t d, int64_t ldw, int64_t ldg,
                            const int32_t* plan, const uint64_t* dest, double lr,
                            unsigned long long* absmax_bits, void* stream,
                                const rm_step_sync* sync);
int rm_ring_mix_sgd_pos_f64(const uint64_t* slot_ptrs, const double* W_local,
                            const double* G_local, int L, int g0, int Lg, int64_t d, int64_t ldw,
                            int64_t ldg, const int32_t* plan, const uint64_t* dest, double lr,
                            unsigned long long* absmax_bits, void* stream,
                                const rm_step_sync* sync);
int rm_ring_mix_sgd_pos_bf16(const uint64_t* slot_ptrs, const uint16_t* W_local,
                             const uint16_t* G_local, int L, int g0, int Lg, int64_t d,
                             int64_t ldw, int64_t ldg, const int32_t* plan, const uint64_t* dest,
                             double lr, unsigned long long* absmax_bits, void* stream,
                                const rm_step_sync* sync);

/* D1D across ranks: S[c] = sum of the local rows (fp64), all-reduced by the
 * caller (NCCL), then out[j] = S/L - lr*G[j]. */
int rm_partial_sum_f32(const float* W, int Lg, int64_t d, int64_t ld, double* S, void* stream);
int rm_partial_sum_f64(const double* W, int Lg, int64_t d, int64_t ld, double* S, void* stream);
int rm_partial_sum_bf16(const uint16_t* W, int Lg, int64_t d, int64_t ld, double* S,
                        void* stream);
int rm_apply_mean_sgd_f32(const double* S, const float* G, float* out, int Lg, int L, int64_t d,
                          int64_t ldg, int64_t ldo, double lr, unsigned long long* absmax_bits,
                          void* stream);
int rm_apply_mean_sgd_f64(const double* S, const double* G, double* out, int Lg, int L,
                          int64_t d, int64_t ldg, int64_t ldo, double lr,
                          unsigned long long* absmax_bits, void* stream);
int rm_apply_mean_sgd_bf16(const double* S, const uint16_t* G, uint16_t* out, int Lg, int L,
                           int64_t d, int64_t ldg, int64_t ldo, double lr,
                           unsigned long long* absmax_bits, void* stream);

/* D1D across ranks through NVSwitch multicast: for columns [c0, c1) sum the
 * ranks' fp64 partial sums in the switch (multimem.ld_reduce) and broadcast the
 * means sum/L to every rank (multimem.st); apply with rm_apply_mean_sgd_*(L = 1).
 * P_mc / M_mc: multicast addresses of symmetric buffers (e.g. torch symmetric
 * memory).  Caller orders it with cross-rank barriers. */
/* Caps, for the calling host thread, on the CTAs per SM launched by rm_partial_sum_* (and
 * rm_column_mean_*), rm_apply_mean_sgd_* and rm_nvls_mean_f64; 0 restores the defaults
 * (16 / 8 / 8).  The D1D training step lowers the first so the average runs beside the
 * gradient generator instead of displacing it.  A chunk
 * pipeline lowers them so the in-switch reduction of one chunk is co-resident (threads and
 * registers) with the local kernels of its neighbours. */
int rm_set_d1d_ctas_per_sm(int partial_sum, int apply, int nvls);
/* Bound, for the calling host thread, on the distinct remote rows a learner-sharded step pulls
 * (0 = the layout's own bound, 2 * Lg).  A fixed ring with contiguous shards pulls at most 2
 * (its boundary neighbours): with the bound the stages hold 1 KB row segments instead of
 * reserving room for 2 * Lg remote rows.  A step whose plan exceeds the bound traps. */
int rm_set_shard_remote_rows(int max_rows);
/* numpy-order learner-sharded D1D, for the calling host thread: `chains` (1, 2, 4, 8; 0 =
 * off) of numpy's eight pairwise chains per rank.  Rank g then holds learners
 * {l : l % 8 in [g chains, (g + 1) chains)} in ascending order (L % 8 == 0, 8 <= L <= 128),
 * rm_partial_sum_* / rm_d1d_fused_* compute numpy's tree over those chains, and the
 * cross-rank sums (rm_p2p_mean_f64, the fused kernels' reduce role) combine ranks in the
 * tree order, so the mean is W.mean(axis=1) bit for bit (mixing.py:122-124) — the sharded
 * step equals the single-GPU step.  Above 2 ranks this needs peer tables (the in-switch
 * sum of more than two addends has no specified order); fp32 / fp64 only. */
int rm_set_d1d_numpy_order(int chains);
/* The learner interleave of the gradient streams of the following rm_quadratic_grad_shard_* /
 * rm_quadratic_mean_step_shard_* calls of this host thread: stream s is learner
 * learner0 + (s / run) * period + s % run (run = 0: learner0 + s). */
int rm_set_shard_streams(int run, int64_t period);
/* D1D across GPUs in ONE launch per rank (simulation.py:304-312 with the learners sharded):
 * the CTAs split into partial-sum / in-switch-reduce / apply roles that walk the column
 * chunks in order and hand chunks to each other (and to the other ranks) through flags.
 *   P, M: symmetric fp64[d] buffers (local addresses) and their multicast addresses;
 *   flags / flags_mc: symmetric uint32[2 * max_chunks], zeroed once on every rank before
 *   the first call; counters: local device uint32[2 * max_chunks], zeroed once;
 *   epoch: 1, 2, 3, ... (one per call, the same on every rank);
 *   chunk_cols: a multiple of 32 * world; pct_partial / pct_reduce: share of the grid's
 *   CTAs for those roles (the rest apply).  Every rank must call with the same d, L,
 *   chunk_cols and epoch.  A wait longer than RINGMIX_XGPU_TIMEOUT_S gives up and is
 *   reported by rm_xgpu_status(). */
int rm_d1d_fused_nvls_f32(const float* W, const float* G, float* out, int Lg, int L, int64_t d,
                          int64_t ldw, int64_t ldg, int64_t ldo, double lr,
                          unsigned long long* absmax_bits, double* P, const double* P_mc,
                          const double* M, double* M_mc, uint32_t* flags, uint32_t* flags_mc,
                          uint32_t* counters, int rank, int world, int64_t chunk_cols,
                          int max_chunks, uint32_t epoch, int pct_partial, int pct_reduce,
                          void* stream);
int rm_d1d_fused_nvls_f64(const double* W, const double* G, double* out, int Lg, int L,
                          int64_t d, int64_t ldw, int64_t ldg, int64_t ldo, double lr,
                          unsigned long long* absmax_bits, double* P, const double* P_mc,
                          const double* M, double* M_mc, uint32_t* flags, uint32_t* flags_mc,
                          uint32_t* counters, int rank, int world, int64_t chunk_cols,
                          int max_chunks, uint32_t epoch, int pct_partial, int pct_reduce,
                          void* stream);
int rm_d1d_fused_nvls_bf16(const uint16_t* W, const uint16_t* G, uint16_t* out, int Lg, int L,
                           int64_t d, int64_t ldw, int64_t ldg, int64_t ldo, double lr,
                           unsigned long long* absmax_bits, double* P, const double* P_mc,
                           const double* M, double* M_mc, uint32_t* flags, uint32_t* flags_mc,
                           uint32_t* counters, int rank, int world, int64_t chunk_cols,
                           int max_chunks, uint32_t epoch, int pct_partial, int pct_reduce,
                           void* stream);
int rm_nvls_mean_f64(const double* P_mc, double* M_mc, int64_t c0, int64_t c1, int L,
                     void* stream);
/* rm_nvls_mean_f64 without multicast: P_peers / M_peers are device uint64[world] tables of
 * every rank's P / M; the cross-rank sum runs in ascending rank order (unicast NVLink
 * loads), the means are stored to every rank. */
int rm_p2p_mean_f64(const uint64_t* P_peers, const uint64_t* M_peers, int world, int64_t c0,
                    int64_t c1, int L, void* stream);

/* The fused D1D step without multicast (unicast NVLink P2P through peer tables), for
 * `nlocal` ranks per launch: 1 in a one-process-per-GPU job on a system without NVSwitch
 * multicast; `world` when every rank's buffers live on this GPU (single-device emulation
 * of the whole world in one launch — what the one-GPU tests run).  ranks: host array of
 * nlocal entries (device pointers inside); P_peers / M_peers / flags_peers: device
 * uint64[world] tables of every rank's P / M / flags.  Cross-rank sums in ascending rank
 * order.  Other arguments as rm_d1d_fused_nvls_*. */
typedef struct {
  const void* W;
  const void* G;
  void* out;
  unsigned long long* absmax_bits;
  double* P;
  const double* M;
  const uint32_t* flags;
  uint32_t* counters;
  int Lg;
  int rank;
} rm_d1d_rank;
int rm_d1d_fused_p2p_f32(const rm_d1d_rank* ranks, int nlocal, int L, int64_t d, int64_t ldw,
                         int64_t ldg, int64_t ldo, double lr, const uint64_t* P_peers,
                         const uint64_t* M_peers, const uint64_t* flags_peers, int world,
                         int64_t chunk_cols, int max_chunks, uint32_t epoch, int pct_partial,
                         int pct_reduce, void* stream);
int rm_d1d_fused_p2p_f64(const rm_d1d_rank* ranks, int nlocal, int L, int64_t d, int64_t ldw,
                         int64_t ldg, int64_t ldo, double lr, const uint64_t* P_peers,
                         const uint64_t* M_peers, const uint64_t* flags_peers, int world,
                         int64_t chunk_cols, int max_chunks, uint32_t epoch, int pct_partial,
                         int pct_reduce, void* stream);
int rm_d1d_fused_p2p_bf16(const rm_d1d_rank* ranks, int nlocal, int L, int64_t d, int64_t ldw,
                          int64_t ldg, int64_t ldo, double lr, const uint64_t* P_peers,
                          const uint64_t* M_peers, const uint64_t* flags_peers, int world,
                          int64_t chunk_cols, int max_chunks, uint32_t epoch, int pct_partial,
                          int pct_reduce, void* stream);

/* ---- device gradient producer for the reference's quadratic oracle ----
 * (objectives.py:84-90 via simulation.py:226-238):
 *   G[l] = lam * (Phi[l] - wopt) + noise_sd * z_l,
 *   z_l = numpy stream(seed, TAG_GRADIENT, k, l).standard_normal(d)   (bit-exact)
 * prefix_words = entropy words of (seed, TAG_GRADIENT); lam/wopt: device fp64[d];
 * Phi/G: learner-major (L, d).  workspace: device, >= rm_normal_workspace_bytes(L, d). */
int64_t rm_normal_workspace_bytes(int nstreams, int64_t n);
/* Larger workspace that also keeps the speculative ziggurat blocks (~8.4 B per
 * normal): with it the output pass is a coalesced copy instead of a re-draw.
 * Any workspace_bytes >= this selects that path; the bits are identical. */
int64_t rm_normal_workspace_bytes_fast(int nstreams, int64_t n);
/* Byte offset inside the workspace of the generator's repair counters
 * (uint32 blocks_rejected_by_merge, uint32 blocks_left_for_sequential_repair). */
int64_t rm_normal_stats_offset(int nstreams, int64_t n);
int rm_quadratic_grad_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k, int L,
                          int64_t d, const float* Phi, int64_t ldp, const double* lam,
                          const double* wopt, double noise_sd, float* G, int64_t ldg,
                          void* workspace, int64_t workspace_bytes, void* stream);
int rm_quadratic_grad_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k, int L,
                          int64_t d, const double* Phi, int64_t ldp, const double* lam,
                          const double* wopt, double noise_sd, double* G, int64_t ldg,
                          void* workspace, int64_t workspace_bytes, void* stream);
/* The same for learners [learner0, learner0 + L) of a learner-sharded run: row l of Phi / G is
 * learner learner0 + l and draws stream(seed, TAG_GRADIENT, k, learner0 + l). */
int rm_quadratic_grad_shard_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                int64_t learner0, int L, int64_t d, const float* Phi, int64_t ldp,
                                const double* lam, const double* wopt, double noise_sd, float* G,
                                int64_t ldg, void* workspace, int64_t workspace_bytes,
                                void* stream);
int rm_quadratic_grad_shard_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                int64_t learner0, int L, int64_t d, const double* Phi,
                                int64_t ldp, const double* lam, const double* wopt,
                                double noise_sd, double* G, int64_t ldg, void* workspace,
                                int64_t workspace_bytes, void* stream);
/* numpy stream(prefix [, k [, s]]).standard_normal(n) for s < nstreams (append = number of
 * trailing entropy ints: 0, 1 = k, 2 = k and the stream index); Z: (nstreams, n) fp64. */
int rm_standard_normal_f64(const uint32_t* prefix_words, int n_prefix, int append, uint64_t k,
                           int nstreams, int64_t n, double* Z, int64_t ldz, void* workspace,
                           int64_t workspace_bytes, void* stream);

/* ---- one training step with the quadratic oracle's gradient fused into the mix ----
 * (simulation.py:263-268 with gradient_matrix simulation.py:226-238 and the oracle
 * objectives.py:84-90):
 *   Wout = apply_mixing(W, T) - lr * G,   G[l] = fl(lam * (Phi[l] - wopt) + noise_sd * z_l)
 * T = the ring given by left/right (randomized or fixed ring), or the uniform matrix when
 * left == right == NULL (D1D).  G is produced inside the mix kernel from the generator's
 * normals and never written: bit-identical to rm_quadratic_grad_* followed by
 * rm_ring_mix_sgd_* / rm_mean_sgd_*.  Phi == NULL (or Phi == W with ldp == ldw) takes the
 * gradient at W itself (synchronous strategies) and reads W once.
 * workspace: device, >= rm_quadratic_mix_workspace_bytes(L, d). */
int64_t rm_quadratic_mix_workspace_bytes(int L, int64_t d);
int rm_quadratic_mix_step_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                              const float* W, const float* Phi, float* Wout, const int32_t* left,
                              const int32_t* right, int L, int64_t d, int64_t ldw, int64_t ldp,
                              int64_t ldo, const double* lam, const double* wopt, double noise_sd,
                              double lr, unsigned long long* absmax_bits, void* workspace,
                              int64_t workspace_bytes, void* stream);
int rm_quadratic_mix_step_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                              const double* W, const double* Phi, double* Wout,
                              const int32_t* left, const int32_t* right, int L, int64_t d,
                              int64_t ldw, int64_t ldp, int64_t ldo, const double* lam,
                              const double* wopt, double noise_sd, double lr,
                              unsigned long long* absmax_bits, void* workspace,
                              int64_t workspace_bytes, void* stream);

/* D1D step of a learner-sharded run with the quadratic oracle's gradient fused in
 * (simulation.py:304-312, objectives.py:84-90): Wout[l] = M - lr * G(Phi[l]) for this rank's
 * learners learner0 + l, l < L, G never written.  M: the global column means (fp64, device),
 * produced concurrently elsewhere (partial sums + cross-GPU reduction on other streams); the
 * generator starts at once and only the final mix waits for `means_ready` (a cudaEvent_t, or
 * NULL).  Same bits as rm_quadratic_grad_shard_* followed by rm_apply_mean_sgd_*(M, G, L=1).
 * workspace: >= rm_quadratic_mix_workspace_bytes(L, d). */
int rm_quadratic_mean_step_shard_f32(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                     int64_t learner0, const double* M, const float* Phi,
                                     float* Wout, int L, int64_t d, int64_t ldp, int64_t ldo,
                                     const double* lam, const double* wopt, double noise_sd,
                                     double lr, unsigned long long* absmax_bits, void* workspace,
                                     int64_t workspace_bytes, void* stream, void* means_ready);
int rm_quadratic_mean_step_shard_f64(const uint32_t* prefix_words, int n_prefix, uint64_t k,
                                     int64_t learner0, const double* M, const double* Phi,
                                     double* Wout, int L, int64_t d, int64_t ldp, int64_t ldo,
                                     const double* lam, const double* wopt, double noise_sd,
                                     double lr, unsigned long long* absmax_bits, void* workspace,
                                     int64_t workspace_bytes, void* stream, void* means_ready);

/* ---- fused trace reductions (run_training's _record, simulation.py:398-409) ----
 * One pass over W (L <= 128 learners, learner-major): cons_sq[l] += sum_c (W[l,c]-mean_c)^2
 * (consensus_distance), and when lam != NULL: loss_col[l] += 0.5 sum_c lam_c (W[l,c]-wopt_c)^2,
 * avg_loss += 0.5 sum_c lam_c (mean_c-wopt_c)^2.  Outputs are fp64 device accumulators the
 * caller zeroes.  Deterministic: CTAs write partials into `workspace` (device,
 * >= rm_trace_stats_workspace_bytes(L)) that a second kernel sums in a fixed order, so the
 * same W gives the same bits on every run (the reference's CSVs are byte-stable). */
int64_t rm_trace_stats_workspace_bytes(int L);
int rm_trace_stats_f32(const float* W, int L, int64_t d, int64_t ld, const double* lam,
                       const double* wopt, double* cons_sq, double* loss_col, double* avg_loss,
                       void* workspace, int64_t workspace_bytes, void* stream);
int rm_trace_stats_f64(const double* W, int L, int64_t d, int64_t ld, const double* lam,
                       const double* wopt, double* cons_sq, double* loss_col, double* avg_loss,
                       void* workspace, int64_t workspace_bytes, void* stream);
int rm_trace_stats_bf16(const uint16_t* W, int L, int64_t d, int64_t ld, const double* lam,
                        const double* wopt, double* cons_sq, double* loss_col, double* avg_loss,
                        void* workspace, int64_t workspace_bytes, void* stream);

/* Exact-order variant (same outputs, WRITTEN rather than accumulated): numpy's own
 * summation order, bit for bit — each learner's sums run sequentially over c like the
 * reference's axis-0 sum and einsum (simulation.py:361, objectives.py:79), the average-model
 * loss is numpy's pairwise sum (objectives.py:72).  d dependent adds per learner
 * (latency-bound): meant for small d (run_training's records, sweeps); any L <= 4096.
 * workspace: device, >= rm_trace_stats_exact_workspace_bytes(d). */
int64_t rm_trace_stats_exact_workspace_bytes(int64_t d);
int rm_trace_stats_exact_f32(const float* W, int L, int64_t d, int64_t ld, const double* lam,
                             const double* wopt, double* cons_sq, double* loss_col,
                             double* avg_loss, void* workspace, int64_t workspace_bytes,
                             void* stream);
int rm_trace_stats_exact_f64(const double* W, int L, int64_t d, int64_t ld, const double* lam,
                             const double* wopt, double* cons_sq, double* loss_col,
                             double* avg_loss, void* workspace, int64_t workspace_bytes,
                             void* stream);
int rm_trace_stats_exact_bf16(const uint16_t* W, int L, int64_t d, int64_t ld,
                              const double* lam, const double* wopt, double* cons_sq,
                              double* loss_col, double* avg_loss, void* workspace,
                              int64_t workspace_bytes, void* stream);

/* Column means M[c] = (numpy pairwise sum over the L learners) / L, fp64, bit-identical
 * to the mean of rm_mean_sgd_*.  With rm_apply_mean_sgd_*(M, G, out, L, 1, ...) it
 * splits the D1D step so the average of W_k runs on a side stream while the
 * gradient of W_{k-1} is produced (north-star (c)). */
int rm_column_mean_f32(const float* W, int L, int64_t d, int64_t ld, double* M, void* stream);
int rm_column_mean_f64(const double* W, int L, int64_t d, int64_t ld, double* M, void* stream);
int rm_column_mean_bf16(const uint16_t* W, int L, int64_t d, int64_t ld, double* M,
                        void* stream);

/* log1p bit-identical to the host glibc 2.39 (x86-64 FMA build), used by the ziggurat tail. */
int rm_log1p_f64(const double* x, double* y, int64_t n, void* stream);

/* ---- batched ring products (monte_carlo_consensus, spectral.py:273-279) ----
 * For b < B: Y_b[j] = ring3(X_b[left_b j], X_b[j], X_b[right_b j]) with `@`
 * (dgemm) rounding, rows of length d at stride ld, batches at batch_stride;
 * left/right are int32[B][L]. */
int rm_ring_mix_batched_f64(const double* X, double* Y, const int32_t* left, const int32_t* right,
                            int B, int L, int64_t d, int64_t ld, int64_t batch_stride,
                            void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RINGMIX_B200_H */
