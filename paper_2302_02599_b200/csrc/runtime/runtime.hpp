// Device runtime: meshes (simulated on one GPU, or one process per GPU over
// NCCL), compiled exchanges and their execution.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../kernels/box_copy.cuh"
#include "../kernels/tile_copy.cuh"
#include "plan.hpp"

namespace apl {

// NVTX range for the lifetime of the object (one per conversion, exchange
// step, all-reduce and sharded matmul; SURVEY §5 tracing). A push/pop pair
// costs a few ns when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name);
  ~NvtxRange();
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Error raised by the runtime; `code` is an apl_status value.
struct RuntimeError : std::runtime_error {
  int code;
  RuntimeError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what);
void check_nccl(ncclResult_t r, const char* what);

FastDiv make_fastdiv(uint32_t d);
int sm_count();
// begins: host copy of the table's unit_begin column (slicing into launches).
cudaError_t launch_box_copy(const DevCopy* d_table, const int64_t* begins, int ntasks,
                            int64_t total_units, int vec_bytes, int max_outer, int max_fan, bool split,
                            const PtrTable& ptrs, cudaStream_t stream,
                            int64_t write_bytes = 0);
// Fused peer exchange: ready-flag announce + acquire, pull, done-flag
// announce in one launch (box_copy.cu, box_pull_sync_kernel).
cudaError_t launch_box_pull_sync(const DevCopy* d_table, const int64_t* begins, int ntasks,
                                 int64_t total_units, int vec_bytes, int max_outer,
                                 const PtrTable& ptrs, const PeerSync& sync, cudaStream_t stream);
cudaError_t launch_allreduce_local(void* const* bufs, const int* members, int groups,
                                   int group_size, size_t count, int dtype,
                                   cudaStream_t stream);
uint64_t launch_count();
cudaError_t launch_gelu_inplace(void* buf, size_t count, int dtype, cudaStream_t stream);
// Fused all-reduce over peer memory (peer_sync.cu / gemm_tcgen05.cu).
cudaError_t launch_peer_allreduce(void* const* members, int P, int64_t count, int dtype,
                                  cudaStream_t stream);
cudaError_t launch_reduce_gather(const float* staging, int P, int64_t slab_elems,
                                 void* const* outs, int nout, bool out_f32, cudaStream_t stream);
cudaError_t gemm_bf16_scatter(const void* A, const void* B, void* const* owner_slabs, int owners,
                              int M, int N, int K, int lda, int ldb, bool b_kn,
                              cudaStream_t stream);
// Peer-exchange epoch flags (peer_sync.cu).
cudaError_t launch_flag_store(uint32_t* const* remote, int n, int slot, uint32_t epoch,
                              cudaStream_t stream);
cudaError_t launch_flag_wait(const uint32_t* flags, const int* slots, int n, uint32_t epoch,
                             uint64_t timeout_ns, cudaStream_t stream);
cudaError_t launch_gelu(const void* x, void* y, size_t count, int dtype, cudaStream_t stream);
cudaError_t launch_gelu_backward(const void* dy, const void* x, void* dx, size_t count, int dtype,
                                 cudaStream_t stream);
// Transformer-block node kinds on one shard (block_ops.cu).
cudaError_t launch_embedding(const int64_t* ids, int64_t n, const void* table, int64_t vocab,
                             int64_t width, int elem_bytes, void* out, cudaStream_t s);
cudaError_t launch_embedding_blocks(const int64_t* ids, int64_t n, const void* const* blocks,
                                    int vocab_blocks, int hidden_blocks, int64_t vocab,
                                    int64_t width, int64_t col_begin, int64_t cols,
                                    int elem_bytes, void* out, cudaStream_t s);
cudaError_t launch_layernorm(const void* x, const void* gamma, const void* beta, void* y,
                             int64_t rows, int64_t width, float eps, int dtype, cudaStream_t s);
cudaError_t launch_softmax(const void* x, void* y, int64_t rows, int64_t width, float alpha,
                           const void* mask, float fill, int dtype, cudaStream_t s);
// any permutation of a row-major tensor of rank <= 8 (y dim d = x dim perm[d])
cudaError_t launch_permute(const void* x, void* y, int rank, const int64_t* shape,
                           const int64_t* perm, int elem_bytes, cudaStream_t s);
// softmax over the middle dim of [outer, len, inner], and its backward
cudaError_t launch_softmax_axis(const void* x, void* y, int64_t outer, int64_t len, int64_t inner,
                                int dtype, cudaStream_t s);
cudaError_t launch_softmax_axis_backward(const void* y, const void* dy, void* dx, int64_t outer,
                                         int64_t len, int64_t inner, float alpha, int dtype,
                                         cudaStream_t s);
cudaError_t launch_transpose(const void* x, void* y, int64_t batch, int64_t rows, int64_t cols,
                             int elem_bytes, cudaStream_t s);
cudaError_t launch_scale(const void* x, void* y, size_t count, float alpha, int dtype,
                         cudaStream_t s);
cudaError_t launch_add(const void* a, const void* b, bool b_mask, void* y, size_t count,
                       float alpha, int dtype, cudaStream_t s);
cudaError_t launch_layernorm_backward(const void* x, const void* gamma, const void* dy, void* dx,
                                      float* dgamma, float* dbeta, void* stats, int64_t rows,
                                      int64_t width, float eps, int dtype, cudaStream_t s);
size_t layernorm_backward_scratch_bytes(int64_t rows, int64_t width);
cudaError_t launch_softmax_backward(const void* y, const void* dy, void* dx, int64_t rows,
                                    int64_t width, float alpha, int dtype, cudaStream_t s);
cudaError_t launch_embedding_backward(const int64_t* ids, int64_t n, const void* dy,
                                      float* dtable, int64_t vocab, int64_t width, int dtype,
                                      cudaStream_t s);
cudaError_t launch_embedding_backward_block(const int64_t* const* ids, const void* const* dy,
                                            int nsrc, int64_t n, int64_t dy_width, float* dblock,
                                            int64_t v0, int64_t rows, int64_t c0, int64_t cols,
                                            int dtype, cudaStream_t s);
cudaError_t launch_mask_not(const void* x, void* y, size_t count, cudaStream_t s);
void gemm_force_plan(int pair, int bn, int streamk);
void gemm_trace(void* buf, size_t bytes);
cudaError_t gemm_bf16(const void* A, const void* B, void* C, int M, int N, int K, int lda,
                      int ldb, int ldc, bool b_kn, bool out_f32, bool gelu, cudaStream_t stream);
cudaError_t gemm_bf16_batched(const void* const* A, const void* const* B, void* const* C,
                              int count, int M, int N, int K, int lda, int ldb, int ldc,
                              bool b_kn, bool out_f32, bool gelu, cudaStream_t stream);

// One sharded-matmul strategy (reference OpStrategy, intraop.hpp:34-49).
struct MatmulStrategy {
  autoplan::ShardingSpec a, b, c;  // on logical A[..m.., k], B[k, n], C[..m.., n]
  bool partial_sum = false;
  std::vector<int> reduce_axes;
};


// A descriptor table resident on the device.
struct CompiledCopies {
  DevCopy* table = nullptr;
  std::vector<int64_t> begins;  // host copy of table[i].unit_begin
  int ntasks = 0;
  int64_t total_units = 0;
  int vec = 16;
  int max_outer = 0;
  int max_fan = 1;
  bool split = false;       // some descriptor has ksplit > 1
  int64_t bytes = 0;        // bytes read (each source byte once)
  int64_t write_bytes = 0;  // bytes written (fan-out counted per destination)
  bool bulk = false;        // TMA bulk engine (units = kBulkSeg segments)
  // TMA tensor-tile engine: the descriptors themselves (tensor maps embed
  // the buffer addresses, so launch arguments are encoded per pointer table
  // and cached for the last table seen).
  bool tile = false;
  std::vector<CopyDesc> tile_descs;
  mutable std::vector<TileArgs> tile_launches;
  mutable PtrTable tile_ptrs{};
  mutable bool tile_cached = false;
  bool empty() const { return ntasks == 0 && tile_descs.empty(); }
};

cudaError_t launch_tile_copy(const TileArgs& args, cudaStream_t stream);
// True when every descriptor suits the tensor-tile engine.
bool tile_eligible(const std::vector<CopyDesc>& descs, int vec);

cudaError_t launch_bulk_copy(const DevCopy* d_table, const int64_t* begins, int ntasks,
                             int64_t total_units, const PtrTable& ptrs, cudaStream_t stream,
                             int64_t write_bytes = 0);
// True when every run of the table suits the TMA bulk engine.
bool bulk_eligible(const std::vector<CopyDesc>& descs, int vec);

// Largest vector width (16/8/4/2/1) dividing every run, stride and offset.
int natural_vec(const std::vector<CopyDesc>& descs);
CompiledCopies compile_copies(const std::vector<CopyDesc>& descs, int vec, bool bulk = false,
                              bool tile = false);
void free_copies(CompiledCopies& c);
void run_copies(const CompiledCopies& c, const PtrTable& ptrs, cudaStream_t stream);

// One direct src -> tgt redistribution, compiled for the local devices.
struct Exchange {
  std::string label;      // NVTX range name: "<kind>|<src>><tgt>" (the cache key)
  int64_t in_bytes = 0;   // per-device source shard bytes
  int64_t out_bytes = 0;  // per-device target shard bytes
  std::vector<CopyDesc> host_copies;  // simulated mesh: everything
  std::vector<CopyDesc> host_pre;     // distributed: pack + self
  std::vector<CopyDesc> host_post;    // distributed: unpack
  std::vector<CopyDesc> host_pull;    // distributed, peer mode: one kernel pulls every
                                      // piece straight from the senders' shards
  std::vector<int> pull_senders;      // peer mode: ranks this rank reads from (not itself)
  std::vector<int> pull_readers;      // peer mode: ranks that read this rank's source
  std::vector<CopyDesc> host_push;    // peer push mode: every piece this rank sends, stored
                                      // straight into the receivers' outputs (dst id = rank)
  std::map<int, CompiledCopies> copies, pre, post, pull, push;  // keyed by vector width
  struct Xfer {
    int peer;
    bool direct;  // straight from `in` / into `out` (contiguous box)
    int64_t offset;
    int64_t bytes;
  };
  std::vector<Xfer> sends, recvs;
  int64_t send_staging = 0, recv_staging = 0;
  int64_t wire_bytes_in = 0;   // bytes this rank receives from peers
  int64_t wire_bytes_out = 0;  // bytes this rank sends to peers
  // Distributed all-gather step (reference kAllGather on one mesh axis):
  // ncclAllGather of the source shard on that axis's communicator into
  // receive staging laid out [n_a][source shard] (group order = coordinate
  // on the axis), then host_post unpacks it into `out`; ag_direct: the
  // gathered layout already is `out` (nothing outside the gathered dim).
  int ag_axis = -1;
  bool ag_direct = false;
  // Distributed all-to-all step (reference kAllToAll on one mesh axis):
  // host_pre packs the n_a equal chunks along the split dim into send
  // staging [n_a][chunk] (skipped when `in` already is that layout),
  // ncclAlltoAll on the axis communicator, host_post unpacks receive staging
  // [n_a][chunk] along the gathered dim (skipped when it lands in `out`).
  int a2a_axis = -1;
  bool a2a_direct_send = false, a2a_direct_recv = false;
  int64_t a2a_chunk = 0;
};


struct Mesh {
  autoplan::DeviceMesh geo;
  int device = 0;
  bool distributed = false;
  int rank = 0;  // distributed: this process's mesh device index
  ncclComm_t world = nullptr;
  std::map<uint32_t, ncclComm_t> sub;  // axis-subset mask -> communicator
  bool aborted = false;                // apl_mesh_abort ran: communicators are gone
  std::mutex mu;
  std::unordered_map<std::string, std::shared_ptr<Exchange>> exchanges;
  // Peer memory: buffers this process allocated for export (true) or opened
  // from another process's IPC handle (false).
  std::map<void*, bool> peer_buffers;

  int num_local() const { return distributed ? 1 : static_cast<int>(geo.num_devices()); }
  ~Mesh();
};

std::shared_ptr<Exchange> get_exchange(Mesh& mesh, const autoplan::ShardingSpec& src,
                                       const autoplan::ShardingSpec& tgt,
                                       const autoplan::TensorMeta& meta);

// Workspace a src -> tgt exchange needs (distributed staging; 0 if simulated).
size_t exchange_workspace(const Exchange& ex);

// Runs `ex` moving in[] -> out[] (num_local pointers each).
void run_exchange(Mesh& mesh, Exchange& ex, const void* const* in, void* const* out,
                  void* ws, size_t ws_bytes, cudaStream_t stream);

// A validated path with its exchanges compiled: one hop when collapsed (or a
// single step), one hop per reference step otherwise (intermediates ping-pong
// through the workspace).
// The all-to-all form of one A2A step on a distributed mesh.
std::shared_ptr<Exchange> get_alltoall(Mesh& mesh, const autoplan::ShardingSpec& src,
                                       const autoplan::TransformStep& step,
                                       const autoplan::TensorMeta& meta);
// The all-gather form of one AG step on a distributed mesh.
std::shared_ptr<Exchange> get_allgather(Mesh& mesh, const autoplan::ShardingSpec& src,
                                        const autoplan::TransformStep& step,
                                        const autoplan::TensorMeta& meta);

struct Conversion {
  Mesh* mesh = nullptr;
  std::vector<std::shared_ptr<Exchange>> hops;
  int64_t inter_bytes = 0;  // per ping-pong region
  int64_t staging = 0;      // distributed pack/unpack staging
};

Conversion prepare_conversion(Mesh& mesh, const autoplan::ShardingSpec& src,
                              const autoplan::ShardingSpec& tgt,
                              const std::vector<autoplan::TransformStep>& steps,
                              const autoplan::TensorMeta& meta, bool fuse);
size_t conversion_workspace(const Conversion& cv);
void run_conversion(Conversion& cv, const void* const* in, void* const* out, void* ws,
                    size_t ws_bytes, cudaStream_t stream);

// Distributed mesh, peer mode: one box-copy launch pulls every piece of this
// rank's target shard straight from the senders' source shards.
// `peer_in[p]` is rank p's source shard mapped into this process (own shard
// at index rank). The caller orders it after every rank's writes to its
// source shard and keeps the sources unchanged until every rank finished.
void run_pull(Mesh& mesh, const autoplan::ShardingSpec& src, const autoplan::ShardingSpec& tgt,
              const autoplan::TensorMeta& meta, const void* const* peer_in, void* out,
              cudaStream_t stream);

// The fused peer exchange in one launch: flags (every rank's flag array
// mapped here, own entry ignored), a zeroed device counter, the epoch.
struct PeerSyncArgs {
  void* const* flags;
  const void* local_flags;
  void* counter;
  uint32_t epoch;
  uint64_t timeout_ns;
};
void run_pull_sync(Mesh& mesh, const autoplan::ShardingSpec& src,
                   const autoplan::ShardingSpec& tgt, const autoplan::TensorMeta& meta,
                   const void* const* peer_in, void* out, const PeerSyncArgs& sync,
                   cudaStream_t stream);
// Peer push: this rank stores every piece it sends straight into the
// receivers' (peer-mapped, exported) outputs -- peer_out[q] = rank q's output
// mapped here, peer_out[rank] = the local output -- in ONE launch that
// announces `epoch` (this rank's output may now be overwritten), acquires the
// announcements of the ranks it writes to, stores, and marks done (slot
// P + rank) at every peer after a system-scope fence. The receiver waits for
// done of its senders (apl_peer_flags_wait) before reading its output.
void run_push_sync(Mesh& mesh, const autoplan::ShardingSpec& src,
                   const autoplan::ShardingSpec& tgt, const autoplan::TensorMeta& meta,
                   const void* in, void* const* peer_out, const PeerSyncArgs& sync,
                   cudaStream_t stream);

size_t path_workspace(Mesh& mesh, const autoplan::ShardingSpec& src,
                      const autoplan::ShardingSpec& tgt,
                      const std::vector<autoplan::TransformStep>& steps,
                      const autoplan::TensorMeta& meta, bool fuse);

void run_path(Mesh& mesh, const autoplan::ShardingSpec& src, const autoplan::ShardingSpec& tgt,
              const std::vector<autoplan::TransformStep>& steps,
              const autoplan::TensorMeta& meta, const void* const* in, void* const* out,
              void* ws, size_t ws_bytes, bool fuse, cudaStream_t stream);

void all_reduce(Mesh& mesh, const std::vector<int>& axes, void* const* bufs, size_t count,
                int dtype, cudaStream_t stream);

// Axis groups of `axes` (reduction groups), members in mixed-radix order.
std::vector<std::vector<int>> axis_groups(const autoplan::DeviceMesh& geo,
                                          const std::vector<int>& axes);

cudaError_t gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                              int groups, int reduce, int fan, int M, int N, int K, int lda,
                              int ldb, int ldc, bool b_kn, bool out_f32, bool gelu,
                              cudaStream_t stream);

// Extended form: A given transposed (a_km: row-major [K, M]) and epilogue
// 0 none / 1 GELU / 2 GELU backward against aux (bf16 [M, N], one per
// output problem).
cudaError_t gemm_bf16_grouped(const void* const* A, const void* const* B, void* const* C,
                              int groups, int reduce, int fan, int M, int N, int K, int lda,
                              int ldb, int ldc, bool b_kn, bool out_f32, int epi, bool a_km,
                              const void* const* aux, int ldaux, cudaStream_t stream);

// B shards are row-major [k_local, n_local] when b_kn, else transposed
// [n_local, k_local] (nn.Linear layout).
// epilogue APL_EPI_GELU_SAVE also stores the pre-activation to aux[d].
void sharded_matmul(Mesh& mesh, const MatmulStrategy& s, const autoplan::TensorMeta& a_meta,
                    const autoplan::TensorMeta& b_meta, const void* const* A,
                    const void* const* B, void* const* C, bool b_kn, int out_dtype,
                    int epilogue, cudaStream_t stream, void* const* aux = nullptr);

// Backward of one strategy: per local device dA = dC . B^T (bf16; with
// dgelu, times GELU'(aux) -- the fused backward of a GELU feeding A) and
// dB = A^T . dC (dB_dtype, in B's storage layout), each summed over the
// mesh axes it is partial over (dA: the axes sharding C's n dim; dB: the
// axes sharding C's m dims). dA / dB may be null to skip.
void sharded_matmul_backward(Mesh& mesh, const MatmulStrategy& s,
                             const autoplan::TensorMeta& a_meta,
                             const autoplan::TensorMeta& b_meta, const void* const* A,
                             const void* const* B, const void* const* dC, void* const* dA,
                             void* const* dB, bool b_kn, bool dgelu, const void* const* aux,
                             int dB_dtype, cudaStream_t stream);

}  // namespace apl
