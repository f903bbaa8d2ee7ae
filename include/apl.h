/* apl.h — C-ABI of the B200 layout-conversion runtime ("autoplan layout").
 *
 * Plain C: fixed-size POD structs, pointers and sizes, int status codes.
 * No exceptions cross this boundary and no CUDA / NCCL / torch types appear
 * in it (streams travel as `void*` = cudaStream_t).
 *
 * What each group replaces in the reference (/root/reference/proj):
 *   spec / path functions  -> ShardingSpec::parse / to_string / valid_for
 *                             (src/layout.cpp:79-160), one_step_transforms
 *                             (layout.cpp:162-221), find_transform_path
 *                             (layout.cpp:253-316), conversion_cost
 *                             (layout.cpp:318-329), PathCache (layout.cpp:331-362),
 *                             collective_cost (src/cluster.cpp:374-400).
 *   runtime functions      -> NEW. The reference only *records* conversions
 *                             (planner.cpp:218-352 CommInsertion / kCommunication
 *                             nodes with name/mesh_axes/axes/bytes attrs); these
 *                             execute them on device data: shard-slice, all-gather,
 *                             all-to-all (CollectiveKind, include/autoplan/
 *                             cluster.hpp:46-52) and the partial-sum all-reduce of
 *                             sharded matmul strategies (intraop.cpp:141-234,
 *                             544-551).
 *
 * Status codes mirror the reference exception hierarchy (errors.hpp:25-108).
 *
 * Data placement: a device at mesh coordinate c holds,
 * for every tensor dim d sharded over axes (a_1..a_m), block index
 * s_d = mixed radix of (c_{a_1}, .., c_{a_m}) with a_1 most significant,
 * stored dense row-major. Mesh coordinates map to device index row-major.
 */
#ifndef APL_H_
#define APL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APL_MAX_DIMS 8  /* tensor rank limit */
#define APL_MAX_MESH 8  /* mesh rank limit */
#define APL_MAX_LOCAL 64 /* simulated devices per local mesh */

typedef enum {
  APL_OK = 0,
  APL_ERR_SCHEMA = 1,     /* SchemaError: malformed spec / mesh text */
  APL_ERR_AXIS = 2,       /* AxisError: mesh axis out of range / reused */
  APL_ERR_SHAPE = 3,      /* ShapeError: spec invalid for tensor/mesh */
  APL_ERR_RANK = 4,       /* RankMismatchError */
  APL_ERR_INFEASIBLE = 5, /* InfeasibleError: no conversion path */
  APL_ERR_CUDA = 6,       /* CUDA runtime failure / no device / no kernel image */
  APL_ERR_NCCL = 7,       /* NCCL failure */
  APL_ERR_ARG = 8,        /* bad argument (null, capacity too small, limits) */
  APL_ERR_PLAN = 9,       /* any other PlanError */
  APL_ERR_INTERNAL = 10   /* anything else */
} apl_status;

/* Same order as autoplan::CollectiveKind (cluster.hpp:46-52). */
typedef enum {
  APL_ALL_GATHER = 0,
  APL_ALL_REDUCE = 1,
  APL_REDUCE_SCATTER = 2,
  APL_ALL_TO_ALL = 3,
  APL_SHARD_SLICE = 4
} apl_kind;

typedef enum { APL_F32 = 0, APL_BF16 = 1, APL_F16 = 2 } apl_dtype;

/* Execution flags for apl_run_path. */
#define APL_STEPWISE 0u   /* run the reference's steps one by one */
#define APL_FUSE_CHAIN 1u /* collapse the whole chain into one exchange pass */

typedef struct {
  int32_t rank;                            /* tensor rank */
  int32_t mesh_rank;
  int32_t naxes[APL_MAX_DIMS];             /* axes per dim (0 = replicated) */
  int32_t axes[APL_MAX_DIMS][APL_MAX_MESH];
} apl_spec;

typedef struct {
  int32_t rank;
  int32_t dtype_bytes; /* 1, 2, 4 or 8 */
  int64_t shape[APL_MAX_DIMS];
} apl_meta;

typedef struct {
  int32_t kind; /* apl_kind */
  int32_t tensor_dim;
  int32_t target_dim; /* all-to-all destination dim, -1 otherwise */
  int32_t mesh_axis;
  apl_spec result;
} apl_step;

/* Per-axis alpha-beta model; NULL alpha/beta arrays select the reference's
 * DeviceMesh::uniform defaults (alpha 1e-5 s, beta_inv 1e-9 s/B). */
typedef struct {
  int32_t ndim;
  int64_t shape[APL_MAX_MESH];
  double alpha[APL_MAX_MESH];
  double beta_inv[APL_MAX_MESH];
} apl_mesh_desc;

/* One exchange piece of a conversion: the box `ext` at `src_lo` of the
 * sender's source shard lands at `dst_lo` of the receiver's target shard
 * (local element coordinates). */
typedef struct {
  int32_t sender;   /* mesh device index (row-major) */
  int32_t receiver; /* mesh device index (row-major) */
  int64_t src_lo[APL_MAX_DIMS];
  int64_t dst_lo[APL_MAX_DIMS];
  int64_t ext[APL_MAX_DIMS];
} apl_piece;

/* ---- diagnostics ---------------------------------------------------- */
int apl_version(void); /* 100 * major + minor */
const char* apl_last_error(void); /* thread-local message of the last failure */

/* ---- spec algebra + path search (host only; no GPU needed) ------------ */
int apl_mesh_desc_uniform(const int64_t* shape, int ndim, apl_mesh_desc* out);
int apl_parse_mesh_shape(const char* text, int64_t* shape, int cap, int* ndim);
/* Mesh documents (reference mesh_to_json / mesh_from_json, cluster.hpp:95-96,
 * cluster.cpp:417-450): to_json writes the reference's five fields with the
 * uniform assignment "d0".."dN-1" (*len = length without the NUL; buf NULL
 * to size); from_json validates like the reference (APL_ERR_SCHEMA on a
 * malformed or inconsistent document) and returns the geometry. */
int apl_mesh_to_json(const apl_mesh_desc* mesh, double device_flops_per_s, char* buf,
                     size_t cap, size_t* len);
int apl_mesh_from_json(const char* text, apl_mesh_desc* out, double* device_flops_per_s);
int apl_spec_parse(const char* text, int mesh_rank, apl_spec* out);
int apl_spec_to_string(const apl_spec* spec, char* buf, size_t cap);
int apl_spec_valid(const apl_spec* spec, const apl_mesh_desc* mesh, const apl_meta* meta,
                   int* valid);
int apl_spec_per_device_bytes(const apl_spec* spec, const apl_mesh_desc* mesh,
                              const apl_meta* meta, int64_t* bytes);
int apl_one_step_transforms(const apl_spec* spec, const apl_mesh_desc* mesh,
                            const apl_meta* meta, apl_step* out, int cap, int* count);
int apl_dim_diff(const int32_t* src_axes, int nsrc, const int32_t* tgt_axes, int ntgt,
                 const double* weights4 /* NULL = defaults {2,1,2,2} */, double* out);
int apl_heuristic_diff(const apl_spec* src, const apl_spec* tgt,
                       const double* weights4, double* out);
int apl_find_transform_path(const apl_mesh_desc* mesh, const apl_spec* src,
                            const apl_spec* tgt, const apl_meta* meta, apl_step* steps,
                            int cap, int* nsteps, double* comm_cost_s);
int apl_collective_cost(const apl_mesh_desc* mesh, const int32_t* axes, int naxes,
                        int kind, double bytes, double* out);

/* PathCache (reference layout.hpp:120-132). Thread safe. */
typedef struct apl_path_cache apl_path_cache;
int apl_path_cache_create(apl_path_cache** out);
int apl_path_cache_destroy(apl_path_cache* cache);
int apl_path_cache_get(apl_path_cache* cache, const apl_mesh_desc* mesh, const apl_spec* src,
                       const apl_spec* tgt, const apl_meta* meta, apl_step* steps, int cap,
                       int* nsteps, double* comm_cost_s);
int apl_path_cache_stats(const apl_path_cache* cache, size_t* searches, size_t* size);
int apl_path_cache_clear(apl_path_cache* cache);

/* Exchange plan of a direct src->tgt redistribution (host only). role 0:
 * pieces `device` receives; role 1: pieces `device` sends. Each target
 * element is sourced exactly once; the sender of a piece is the source
 * replica that agrees with the receiver on every axis the source spec does
 * not use, so traffic stays inside the source's axis groups and a device
 * never receives bytes it already holds. */
int apl_plan_pieces(const apl_mesh_desc* mesh, const apl_spec* src, const apl_spec* tgt,
                    const apl_meta* meta, int device, int role, apl_piece* out, int cap,
                    int* count);

/* ---- runtime (CUDA) --------------------------------------------------- */
typedef struct apl_mesh apl_mesh;

/* Simulated mesh: every mesh device is a separate buffer on one GPU (the
 * 1-GPU parity / HBM-roofline mode). Buffer arrays passed to the run
 * functions then hold num_devices pointers in row-major device order. */
int apl_mesh_create_local(const apl_mesh_desc* mesh, int cuda_device, apl_mesh** out);

/* Distributed mesh: one process per GPU. `nccl_id` is 128 bytes made by
 * apl_nccl_unique_id on rank 0 and broadcast by the caller. Buffer arrays
 * then hold exactly one pointer (this rank's shard). Builds one NCCL
 * sub-communicator per non-empty mesh-axis subset (ncclCommSplit, color =
 * coordinates off the subset, key = coordinates on it). */
int apl_nccl_unique_id(uint8_t* out128);
int apl_mesh_create_nccl(const apl_mesh_desc* mesh, int rank, const uint8_t* nccl_id,
                         int cuda_device, apl_mesh** out);
int apl_mesh_destroy(apl_mesh* mesh);

/* Failure detection for NCCL meshes (the reference has no
 * runtime): polls ncclCommGetAsyncError on the world and every axis-subset
 * communicator. *state = 0 healthy, 7 (ncclInProgress) an operation still
 * completing, else the first ncclResult_t error. Simulated and peer meshes
 * report 0. apl_mesh_abort runs ncclCommAbort on every communicator (after a
 * timeout or an async error): pending NCCL kernels return, the mesh becomes
 * unusable (later NCCL calls fail with APL_ERR_NCCL) and destroy skips
 * ncclCommDestroy. */
int apl_mesh_health(apl_mesh* mesh, int* state);
int apl_mesh_abort(apl_mesh* mesh);

/* Distributed mesh over peer memory only (no NCCL): the transport is CUDA
 * IPC-mapped peer pointers (NVLink through NVSwitch between GPUs; also valid
 * between processes sharing one GPU). Used by apl_run_pull. */
int apl_mesh_create_peer(const apl_mesh_desc* mesh, int rank, int cuda_device, apl_mesh** out);

/* Device buffer exported to the other ranks: cudaMalloc'd (an allocation
 * base, as IPC requires) plus its 64-byte IPC handle. Freed with the mesh. */
int apl_peer_alloc(apl_mesh* mesh, size_t bytes, void** ptr, uint8_t* handle64);
/* Maps another process's exported buffer; closed with the mesh. */
int apl_peer_open(apl_mesh* mesh, const uint8_t* handle64, void** ptr);

/* Device-side epoch flags for peer exchanges without host barriers. Every
 * rank owns a uint32 flag array of 2 x num_ranks entries (apl_peer_alloc +
 * zero fill; peers map it with apl_peer_open). apl_peer_flags_store writes
 * `epoch` into entry `slot` of each of the n mapped arrays (system-scope
 * release after a system fence; stream-ordered after the work it announces).
 * apl_peer_flags_wait blocks the stream until local_flags[slots[i]] >= epoch
 * for all i (acquire; traps with a launch error after timeout_ms instead of
 * hanging). Protocol at epoch e on rank r (see PeerMesh.exchange_async):
 * store ready (slot r) -> wait ready of the senders -> apl_run_pull -> store
 * done (slot P + r); before overwriting the source: wait done of the readers. */
int apl_peer_flags_store(void* const* remote_flags, int n, int slot, uint32_t epoch,
                         void* stream);
int apl_peer_flags_wait(const void* local_flags, const int32_t* slots, int n, uint32_t epoch,
                        uint32_t timeout_ms, void* stream);

/* Fused split-k GEMM + all-reduce over peer memory (Megatron fc2 /
 * split-k strategies on a peer mesh group of P <= 8 ranks), two kernels:
 *  apl_peer_gemm_scatter: C_r = A . B (bf16 in, fp32 partial) with row block
 *    q of the partial stored straight into owner q's staging slab for this
 *    rank (owner_slabs[q], peer-mapped): the reduce-scatter's transfer is
 *    the GEMM epilogue, overlapping the next tiles' MMAs. M / P must be a
 *    multiple of 128.
 *  apl_peer_reduce_gather: the owner sums its P received slabs (rank order)
 *    and writes the result into every rank's output rows (outs[q], peer-
 *    mapped): the all-gather as peer stores. Every replica is bit-identical.
 * Ordering between the two (and across epochs) uses apl_peer_flags_*. */
int apl_peer_gemm_scatter(const void* A, const void* B, void* const* owner_slabs, int owners,
                          int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb,
                          int b_layout, void* stream);
int apl_peer_reduce_gather(const float* staging, int P, int64_t slab_elems, void* const* outs,
                           int nout, int out_dtype, void* stream);

/* In-place all-reduce over peer memory, ONE kernel per rank: members[r] =
 * member r's buffer at this rank's block (count elements, 16-byte aligned,
 * f32 or bf16). The owner of each block sums it over the members in member
 * order (fp32) and writes the sum back to every member; blocks of different
 * owners are disjoint. Bracket with apl_peer_flags_* (ready before, done
 * after). Used for partial sums over arbitrary mesh-axis groups. */
int apl_peer_allreduce(void* const* members, int P, size_t count, int dtype, void* stream);

/* Fused collapsed exchange over peer memory: ONE kernel pulls every piece of
 * this rank's target shard straight out of the senders' source shards
 * (peer_in[r] = rank r's source shard mapped into this process, this rank's
 * own shard at index rank) and writes it in place — no pack, no staging, no
 * separate collective. The caller orders it after all ranks' writes to their
 * source shards and keeps them unchanged until every rank has pulled. */
int apl_run_pull(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt, const apl_meta* meta,
                 const void* const* peer_in, void* out, void* stream);

/* The same exchange with its ordering fused in: ONE launch per exchange.
 * CTA 0 stores `epoch` into slot `rank` of every peer's flag array (this
 * rank's source is ready), every CTA waits (acquire, system scope, trap after
 * timeout_ms) until the ranks it actually reads from announced `epoch`, the
 * pull runs, and the last CTA stores `epoch` into slot P + rank of every
 * peer's array (done reading). peer_flags[q] = rank q's flag array mapped
 * here (own entry unused); counter = a zeroed 4-byte device word used by
 * one exchange at a time (stream-serial). Before overwriting its source the
 * caller waits for `done` of the ranks apl_exchange_peers lists as readers
 * (apl_peer_flags_wait). Replaces the store/wait/pull/store sequence. */
typedef struct {
  void* const* peer_flags;
  const void* local_flags;
  void* counter;
  uint32_t epoch;
  uint32_t timeout_ms;
} apl_peer_sync;
int apl_run_pull_sync(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                      const apl_meta* meta, const void* const* peer_in, void* out,
                      const apl_peer_sync* sync, void* stream);
/* The same exchange as a PUSH (remote stores instead of remote loads): this
 * rank stores every piece it sends straight into the receivers' outputs.
 * peer_out[q] = rank q's output mapped here (exported memory), peer_out[rank]
 * = the local output; in = this rank's source (local). One launch: CTA 0
 * stores `epoch` into slot `rank` of every peer (this rank's output may be
 * overwritten), every CTA waits until the ranks it writes to announced
 * `epoch`, the stores run, and after a system-scope fence the last CTA
 * stores `epoch` into slot P + rank of every peer (done writing). The
 * receiver waits for done of its senders (apl_exchange_peers' `senders`,
 * apl_peer_flags_wait on slots P + s) before reading its output; the source
 * is never read remotely, so no wait is needed before overwriting it. */
int apl_run_push_sync(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                      const apl_meta* meta, const void* in, void* const* peer_out,
                      const apl_peer_sync* sync, void* stream);
/* Peers of this rank in a src -> tgt peer exchange: the ranks it reads from
 * (senders) and the ranks that read its source (readers); arrays of
 * num_devices entries (either may be NULL to count only). */
int apl_exchange_peers(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                       const apl_meta* meta, int32_t* senders, int* n_senders, int32_t* readers,
                       int* n_readers);
int apl_mesh_info(const apl_mesh* mesh, int* num_devices, int* first_local, int* num_local,
                  int* is_distributed);

/* Workspace needed by apl_run_path / apl_run_step for these arguments. */
int apl_path_workspace_bytes(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                             const apl_step* steps, int nsteps, const apl_meta* meta,
                             unsigned flags, size_t* bytes);

/* Execute one reference TransformStep: out = step applied to in. */
int apl_run_step(apl_mesh* mesh, const apl_spec* src, const apl_step* step,
                 const apl_meta* meta, const void* const* in, void* const* out, void* ws,
                 size_t ws_bytes, void* stream);

/* Execute a TransformPath: stepwise, or collapsed into one exchange when
 * flags has APL_FUSE_CHAIN. Stream ordered; in/out must not alias. */
int apl_run_path(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                 const apl_step* steps, int nsteps, const apl_meta* meta,
                 const void* const* in, void* const* out, void* ws, size_t ws_bytes,
                 unsigned flags, void* stream);

/* Algorithmic traffic of the collapsed src->tgt exchange for this mesh's
 * local devices: bytes the copy kernels read (each source byte once) and
 * write (every destination), and bytes received from other mesh devices
 * (what crosses NVLink on a distributed mesh). */
int apl_exchange_traffic(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                         const apl_meta* meta, int64_t* hbm_read, int64_t* hbm_write,
                         int64_t* wire_in);

/* Copy engine the collapsed src->tgt exchange runs on (16-byte aligned
 * buffers): 0 = vectorised LDG/STG box copy, 1 = TMA bulk engine, 2 = TMA
 * tensor-tile engine. */
int apl_exchange_engine(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                        const apl_meta* meta, int* engine);

/* Host-only dry run of the distributed executor: the exact schedule rank
 * `rank` would run for the collapsed src->tgt exchange (pack/self copies,
 * NCCL sends/recvs with their staging offsets, unpack copies) as JSON.
 * Used to check the N>1 path on CPU (tests/test_distributed_gloo.py). */
int apl_exchange_schedule_json(const apl_mesh_desc* mesh, int rank, const apl_spec* src,
                               const apl_spec* tgt, const apl_meta* meta, char* out, size_t cap,
                               size_t* len);
/* Host-only dry run of a whole conversion for `rank` of a distributed mesh:
 * {"hops": [schedule of each hop, as apl_exchange_schedule_json, plus
 * "allgather": {"axis", "direct"} for hops that are one all-gather on an axis
 * communicator], "inter_bytes", "staging"} -- what apl_run_path executes
 * with `flags` (APL_FUSE_CHAIN / APL_STEPWISE) on an NCCL mesh. */
int apl_conversion_schedule_json(const apl_mesh_desc* mesh, int rank, const apl_spec* src,
                                 const apl_spec* tgt, const apl_step* steps, int nsteps,
                                 const apl_meta* meta, unsigned flags, char* out, size_t cap,
                                 size_t* len);

/* Prepared conversion: validates the path and compiles its exchanges once,
 * so the per-call cost is one lookup-free launch sequence (and the calls can
 * be captured into a CUDA graph after the first run). Same semantics as
 * apl_run_path. */
typedef struct apl_conversion apl_conversion;
int apl_conversion_create(apl_mesh* mesh, const apl_spec* src, const apl_spec* tgt,
                          const apl_step* steps, int nsteps, const apl_meta* meta,
                          unsigned flags, apl_conversion** out);
int apl_conversion_workspace(const apl_conversion* conv, size_t* bytes);
int apl_conversion_run(apl_conversion* conv, const void* const* in, void* const* out, void* ws,
                       size_t ws_bytes, void* stream);
int apl_conversion_destroy(apl_conversion* conv);

/* Sum partial results over the mesh axes `axes` (partial_sum strategies,
 * intraop.cpp:544-551; planner.cpp:263-282). In place; every member of an
 * axis group ends with identical bytes. */
int apl_all_reduce(apl_mesh* mesh, const int32_t* axes, int naxes, void* const* bufs,
                   size_t count, int dtype, void* stream);

/* ---- sharded matmul strategies (reference intraop.cpp:141-234) -------- */
#define APL_EPI_NONE 0
#define APL_EPI_GELU 1 /* exact erf GELU, applied after any partial-sum reduction */
#define APL_EPI_GELU_SAVE 3 /* GELU, and the pre-activation kept in aux (training) */

/* One SPMD matmul strategy of the reference catalog: C[..m.., n] = A[..m.., k]
 * . B[k, n]; specs are on the LOGICAL tensors exactly as the reference writes
 * them (OpStrategy, intraop.hpp:34-49). partial_sum strategies (split-k
 * forms) all-reduce C over reduce_axes. */
typedef struct {
  apl_spec a;
  apl_spec b;
  apl_spec c;
  int32_t partial_sum;
  int32_t nreduce;
  int32_t reduce_axes[APL_MAX_MESH];
} apl_matmul_strategy;

/* Strategy catalog entry (reference OpStrategy, intraop.hpp:34-49). */
typedef struct {
  char name[64];
  apl_matmul_strategy strategy;
  double compute_time_s, comm_time_s, bwd_compute_time_s, bwd_comm_time_s;
  int64_t comm_buffer_bytes, memory_bytes;
} apl_strategy_info;

/* Every valid strategy of a matmul (batched = 0) or batched matmul on the
 * mesh, in the reference catalog's order (intraop.cpp:141-234, 497-555). */
int apl_matmul_strategies(const apl_mesh_desc* mesh, const apl_meta* a_meta,
                          const apl_meta* b_meta, int batched, double device_flops_per_s,
                          apl_strategy_info* out, int cap, int* count);

/* Physical layout of the B operand. */
#define APL_B_NK 0 /* Bt [N, K], K contiguous (nn.Linear weight layout) */
#define APL_B_KN 1 /* B [K, N], N contiguous (the logical reference layout) */

/* Local dense contraction on the tcgen05 tensor cores:
 * C[M,N] = epi(A[M,K] . B[K,N]); A bf16 with unit stride along K, B bf16 in
 * either layout (b_layout), fp32 accumulation in TMEM, C bf16 or f32. */
int apl_gemm_bf16(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                  int64_t lda, int64_t ldb, int64_t ldc, int b_layout, int out_dtype,
                  int epilogue, void* stream);
/* Force parts of every later GEMM's launch plan (-1 = automatic): pair != 0
 * the 2-CTA kernel (256-row tiles), bn the N tile (128 / 256), streamk 1 the
 * stream-K schedule, 2..4 aligned split-K by that factor (each unit one K
 * slice of one tile). For A/B measurements; results do not change beyond
 * fp32 summation order. */
int apl_gemm_force_plan(int pair, int bn, int streamk);

/* Diagnostics: CTA-pair GEMM launches write per-CTA phase timestamps into the
 * device buffer `buf` of `bytes` bytes (16 u64 per CTA: slot 0 %globaltimer at
 * entry; slots 1, 2, 3, 6-11 %clock64 at entry, after the prologue, after
 * griddepcontrol.wait, last accumulator committed, last accumulator drained,
 * last store issued, bulk stores done, teardown, exit; nothing is stamped
 * inside the K loop). A launch with more CTAs than `bytes` holds runs
 * untraced. NULL turns it off. Not for production launches: every traced
 * launch copies the argument block once more. APL_ERR_ARG when `bytes` is
 * below one CTA's 128. */
int apl_gemm_trace(void* buf, size_t bytes);

/* Grouped GEMM, one persistent launch: `groups` output problems, each the
 * sum over `reduce` inputs C_g = epi(sum_r A[g*reduce+r] . B[g*reduce+r]),
 * all problems [M,N] with inner dim K and the given leading dimensions.
 * With reduce > 1 this is an all-gather of the B operand fused into the
 * GEMM: the K-slices of a gathered weight are read straight from the
 * buffers (or peer-mapped shards) that own them, no gathered copy. aux:
 * APL_EPI_GELU_SAVE / APL_EPI_DGELU buffers, one per group (else NULL). */
int apl_gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                          int groups, int reduce, int64_t M, int64_t N, int64_t K, int64_t lda,
                          int64_t ldb, int64_t ldc, int b_layout, int out_dtype, int epilogue,
                          const void* const* aux, void* stream);

/* Execute a strategy on the mesh: per local device one tcgen05 GEMM on its
 * shards (A: local shard of A; B: local shard of B, [k_local, n_local] for
 * APL_B_KN or transposed [n_local, k_local] for APL_B_NK; C: local shard of
 * C), then the partial-sum all-reduce over reduce_axes, then the epilogue if
 * it could not be fused. */
int apl_sharded_matmul(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                       const apl_meta* a_meta, const apl_meta* b_meta, const void* const* A,
                       const void* const* B, void* const* C, int b_layout, int out_dtype,
                       int epilogue, void* stream);

/* apl_sharded_matmul with an aux buffer per local device: APL_EPI_GELU_SAVE
 * (bf16 C) writes GELU(acc) to C and the pre-activation acc to aux -- one
 * pass over the tile for a training forward that needs both. */
int apl_sharded_matmul_ex(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                          const apl_meta* a_meta, const apl_meta* b_meta, const void* const* A,
                          const void* const* B, void* const* C, int b_layout, int out_dtype,
                          int epilogue, void* const* aux, void* stream);

/* Exact-erf GELU in place over `count` elements (elementwise-unary nodes of
 * a plan that could not be fused into a GEMM epilogue). */
int apl_gelu_inplace(void* buf, size_t count, int dtype, void* stream);

/* ---- backward (reverse-path conversions + gradient sync) ---
 * The reference prices the backward pass (reverse-path conversions,
 * ckpt.cpp:348-356; gradient all-reduce over replica axes, ckpt.cpp:359-395,
 * planner.cpp:358-385) but never runs it. These entry points execute it. */

/* y = GELU(x) out of place (a training forward keeps the pre-activation). */
int apl_gelu(const void* x, void* y, size_t count, int dtype, void* stream);
/* dx = dy * GELU'(x). */
int apl_gelu_backward(const void* dy, const void* x, void* dx, size_t count, int dtype,
                      void* stream);

/* ---- transformer-block node kinds (gpt_block plans) -------
 * The non-GEMM kinds of the reference's block graph (graph_ir.cpp:40-46,
 * shape rules graph_ir.cpp:240-345) on ONE device's shard. Every strategy
 * the reference generates for them is local (intraop.cpp:280-450), so these
 * never communicate; the plan executor converts their inputs first. dtype:
 * APL_F32 or APL_BF16, fp32 math. */

/* embedding-lookup: out[t, :] = table[ids[t], :] for n int64 ids; table
 * [vocab, width] of elem_bytes elements (a hidden-sharded table is just a
 * narrower one). Ids outside [0, vocab) give zero rows. */
int apl_embedding_lookup(const int64_t* ids, int64_t n, const void* table, int64_t vocab,
                         int64_t width, int elem_bytes, void* out, void* stream);
/* embedding-lookup with the table's all-gather fused in: the table
 * [vocab, width] is given as its owners' blocks, a row-major grid of
 * vocab_blocks x hidden_blocks (<= 64) equal contiguous blocks [vocab /
 * vocab_blocks, width / hidden_blocks] (a simulated mesh's shards or
 * peer-mapped shards, e.g. a vocab-sharded `src:S0R` table consumed
 * replicated, gpt_block `wte`). out [n, cols] = table[ids, col_begin :
 * col_begin + cols], read in place; no gathered copy of the table. */
int apl_embedding_lookup_blocks(const int64_t* ids, int64_t n, const void* const* blocks,
                                int vocab_blocks, int hidden_blocks, int64_t vocab, int64_t width,
                                int64_t col_begin, int64_t cols, int elem_bytes, void* out,
                                void* stream);
/* layernorm over the last dim: y = (x - mean) / sqrt(var + eps) * gamma + beta
 * per row of `width`; gamma / beta may be NULL (no affine). */
int apl_layernorm(const void* x, const void* gamma, const void* beta, void* y, int64_t rows,
                  int64_t width, float eps, int dtype, void* stream);
/* softmax over the last dim (rows of `width`). */
int apl_softmax(const void* x, void* y, int64_t rows, int64_t width, int dtype, void* stream);
/* softmax(alpha * x + fill * mask) over the last dim: the attention
 * scale -> additive-mask -> softmax chain of the block graph (scaled, att_in,
 * att) in one pass when the plan keeps the three in one layout. mask: u8
 * [rows, width] or NULL. */
int apl_softmax_ex(const void* x, void* y, int64_t rows, int64_t width, float alpha,
                   const void* mask, float fill, int dtype, void* stream);
/* transpose perm [0, 2, 1]: x [batch, rows, cols] -> y [batch, cols, rows]. */
int apl_transpose(const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                  int elem_bytes, void* stream);
/* any transpose: x row-major with extents shape[0..rank) (rank <= 8), y the
 * row-major tensor with y dim d = x dim perm[d] (graph_ir.cpp:270-290).
 * Out of place; bit-exact element moves (elem_bytes 1/2/4/8). */
int apl_permute(const void* x, void* y, int rank, const int64_t* shape, const int64_t* perm,
                int elem_bytes, void* stream);
/* softmax over the middle dim of a row-major [outer, len, inner] tensor (the
 * graph's softmax `axis` when it is not the last), and its backward from the
 * output: dx = alpha * y * (dy - sum_axis(dy * y)). */
int apl_softmax_axis(const void* x, void* y, int64_t outer, int64_t len, int64_t inner,
                     int dtype, void* stream);
int apl_softmax_axis_backward(const void* y, const void* dy, void* dx, int64_t outer,
                              int64_t len, int64_t inner, float alpha, int dtype, void* stream);
/* elementwise-unary y = alpha * x. */
int apl_scale(const void* x, void* y, size_t count, float alpha, int dtype, void* stream);
/* elementwise-binary y = a + alpha * b; b has a's dtype, or with b_mask != 0
 * is a u8 0/1 mask (alpha = -1e4: the additive attention mask). */
int apl_add(const void* a, const void* b, int b_mask, void* y, size_t count, float alpha,
            int dtype, void* stream);
/* elementwise-unary on a u8 mask: y = !x. */
int apl_mask_not(const void* x, void* y, size_t count, void* stream);

/* Backward of the block kinds (the training step of a gpt_block plan). */
/* layernorm: dx; with dgamma / dbeta (fp32 [width], ACCUMULATED: +=) also the
 * affine gradients, which need `stats` scratch of
 * apl_layernorm_backward_scratch() bytes (16-byte aligned). The affine
 * gradients are reduced without atomics: bit-reproducible. */
int apl_layernorm_backward_scratch(int64_t rows, int64_t width, size_t* bytes);
int apl_layernorm_backward(const void* x, const void* gamma, const void* dy, void* dx,
                           float* dgamma, float* dbeta, void* stats, int64_t rows, int64_t width,
                           float eps, int dtype, void* stream);
/* The same with the scratch size passed in (apl_version >= 101): returns
 * APL_ERR_ARG instead of writing past `stats` when stats_bytes is below
 * apl_layernorm_backward_scratch(). */
int apl_layernorm_backward_ex(const void* x, const void* gamma, const void* dy, void* dx,
                              float* dgamma, float* dbeta, void* stats, size_t stats_bytes,
                              int64_t rows, int64_t width, float eps, int dtype, void* stream);
/* softmax (last dim) from its output y: dx = alpha * y * (dy - sum(dy * y)). */
int apl_softmax_backward(const void* y, const void* dy, void* dx, int64_t rows, int64_t width,
                         float alpha, int dtype, void* stream);
/* embedding: dtable[ids[t], :] += dy[t, :] (fp32 table gradient, accumulated).
 * Deterministic: the (id, token) keys are radix-sorted, each distinct id's
 * tokens are summed in ascending token order by one warp and added to its
 * row once -- no float atomics, the same bytes on every run. Scratch comes
 * from the stream-ordered allocator (cudaMallocAsync). */
int apl_embedding_backward(const int64_t* ids, int64_t n, const void* dy, float* dtable,
                           int64_t vocab, int64_t width, int dtype, void* stream);

/* embedding backward with the gradient's reduce-scatter fused in (same
 * deterministic id-sorted accumulation, tokens ordered by (source, token)): the block
 * [rows, cols] of the table gradient at vocab rows [v0, v0 + rows) and columns
 * [c0, c0 + cols) accumulates (+=, fp32) the rows of every source s -- ids[s]
 * (n int64) with their output gradients dy[s] ([n, dy_width]) -- whose id
 * falls in the block. One call per owner block replaces a per-device
 * [vocab, width] partial gradient + all-reduce + slice. */
int apl_embedding_backward_block(const int64_t* const* ids, const void* const* dy, int nsrc,
                                 int64_t n, int64_t dy_width, float* dblock, int64_t v0,
                                 int64_t rows, int64_t c0, int64_t cols, int dtype, void* stream);

/* Physical layout of the A operand. */
#define APL_A_MK 0 /* A [M, K], K contiguous */
#define APL_A_KM 1 /* A stored transposed, row-major [K, M] (an activation read as A^T) */
/* Grouped tcgen05 GEMM with both operand layouts: C_g = A_g . B_g for
 * `groups` equally shaped problems (batched matmul forward and backward). */
int apl_gemm_bf16_grouped_ex(const void* const* A, const void* const* B, void* const* C,
                             int groups, int64_t M, int64_t N, int64_t K, int64_t lda,
                             int64_t ldb, int64_t ldc, int a_layout, int b_layout, int out_dtype,
                             void* stream);

#define APL_EPI_DGELU 2 /* backward epilogue: dA *= GELU'(aux) */

/* Backward of apl_sharded_matmul for the same strategy and shards: per local
 * device dA = dC . B^T (bf16, [m_local, k_local]; epilogue APL_EPI_DGELU
 * multiplies by GELU'(aux), aux = the bf16 pre-activation that produced A)
 * and dB = A^T . dC (dB_dtype, in B's storage layout b_layout). Each is
 * summed over the mesh axes it is partial over: dA over the axes sharding
 * C's n dim, dB over the axes sharding C's m dims (the data-parallel
 * gradient all-reduce). dA or dB may be NULL. dC must be the (replicated)
 * gradient of the all-reduced C. */
int apl_sharded_matmul_backward(apl_mesh* mesh, const apl_matmul_strategy* strategy,
                                const apl_meta* a_meta, const apl_meta* b_meta,
                                const void* const* A, const void* const* B,
                                const void* const* dC, void* const* dA, void* const* dB,
                                int b_layout, int dA_epilogue, const void* const* aux,
                                int dB_dtype, void* stream);

/* Kernel launches this process issued through the library (evidence). */
int apl_launch_count(uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* APL_H_ */
