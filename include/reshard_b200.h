/* reshard_b200.h — C ABI of the B200-native PTC reshard path (drop-in boundary).
 *
 * The reference (arxiv 2312.05181 "Tenplex"; /root/reference) is a C++20 library,
 * namespace `reshard`, with no FFI of its own.  These entry points are the flat C binding a
 * maintainer would put in front of it (ctypes / cgo / JNI), one per reference operation:
 *
 *   rs_slice / _host         reshard::slice             proj/include/reshard/tensor/tensor.hpp:42
 *                                                        proj/src/tensor/tensor.cpp:61-78
 *   rs_merge / _host         reshard::merge             tensor.hpp:47, tensor.cpp:80-114
 *   rs_range_parse/_format   Range::parse / to_string   range.hpp:59-60, range.cpp:92-144
 *   rs_grid_cells            SplitGrid::cells           split_grid.hpp:37, split_grid.cpp:62-86
 *   rs_grid_refine           grid_refine                split_grid.hpp:55, split_grid.cpp:119-130
 *   rs_even_split            SplitGrid::even_split      split_grid.hpp:23, split_grid.cpp:9-18
 *   rs_errc_name             errc_name                  proj/include/reshard/error.hpp:50, error.cpp:5-41
 *   rs_fnv1a64               fnv1a64                    proj/include/reshard/util/hash.hpp:42
 *   rs_build_strategy        build_strategy
 *   rs_hosted_subtensors     hosted_subtensors
 *   rs_validate              validate
 *   rs_generate_plan         generate_plan              SPEC.md:224-234 (Alg. 1)
 *   rs_recover               recover
 *   rs_plan_cost / _text     plan_cost / serialization
 *   rs_executor_*            apply_plan (distributed)
 *
 * Conventions.  Every int-returning call returns 0 on success, else 1 + errc where errc is
 * the reference's `enum class Errc` value (error.hpp:8-48, numbering unchanged) or one of
 * the codes appended after ScriptError (RS_ERRC_CUDA ...).  rs_last_error() returns the
 * thread's last message, formatted "<ErrcName>: <detail>" like reshard::Error::what()
 * (error.hpp:55-56).  No C++ exception crosses this boundary.  Device pointers are plain
 * CUDA device addresses; the caller owns all payload buffers, handles own descriptors,
 * streams and events.  There is no CPU fallback: without a GPU the device calls fail with
 * RS_ERRC_DEVICE_UNAVAILABLE.
 */
#ifndef RESHARD_B200_H
#define RESHARD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_MAX_RANK 8

/* error codes (errc values; the call's return is 1 + errc) */
#define RS_ERRC_CHECKPOINT_REQUIRED 28
#define RS_ERRC_SCRIPT_ERROR 31
#define RS_ERRC_CUDA 32
#define RS_ERRC_DEVICE_UNAVAILABLE 33
#define RS_ERRC_INVALID_ARGUMENT 34

/* dtype codes: reference Dtype (dtype.hpp:12-17) plus BF16 (2-byte opaque payload) */
enum rs_dtype { RS_F32 = 0, RS_F16 = 1, RS_I64 = 2, RS_U8 = 3, RS_BF16 = 4 };

/* state kinds of the GPT catalog preset */
enum rs_state_kind { RS_FP32_ADAM = 0, RS_MIXED_ADAM = 1, RS_FP32_PARAM = 2 };

/* layer tags of catalog entries that are not in a transformer layer */
#define RS_LAYER_PRE (-1)
#define RS_LAYER_POST (-2)

typedef struct rs_range {
  int32_t rank;
  uint64_t lo[RS_MAX_RANK];
  uint64_t hi[RS_MAX_RANK];
} rs_range;

typedef struct rs_tensor {  /* a dense row-major tensor in device memory */
  int32_t dtype;
  int32_t rank;
  uint64_t shape[RS_MAX_RANK];
  const void* data;
} rs_tensor;

typedef struct rs_device {
  uint32_t worker;
  uint32_t local;
} rs_device;

typedef struct rs_plan_stats {
  uint64_t n_split, n_move, n_merge;
  uint64_t moved_bytes;    /* sum of Move bytes */
  uint64_t relayout_bytes; /* resident fragments copied into a re-shaped cell */
  uint64_t kept_bytes;     /* resident cells reused in place */
  uint64_t dst_bytes;      /* all destination cells */
} rs_plan_stats;

typedef struct rs_timing {
  float ms;                /* CUDA-event time of the copy kernel on its launch stream */
  uint64_t tiles;
  uint64_t bytes;          /* algorithmic bytes written by this GPU */
  uint64_t launches;       /* kernels launched in the timed region */
  uint64_t read_bytes;     /* algorithmic bytes read (fan-out tiles read their source once) */
  float main_ms;           /* CUDA-event time of the dominant kernel alone, 0 if not timed
                              separately (rs_repartition: the gather pass) */
} rs_timing;

typedef struct rs_cell_binding {
  int32_t gpu;             /* world GPU index */
  int32_t arena;           /* 0: src arena, 1: dst arena */
  uint64_t offset;
  uint64_t bytes;
} rs_cell_binding;

typedef struct rs_context rs_context;
typedef struct rs_catalog rs_catalog;
typedef struct rs_ptc rs_ptc;
typedef struct rs_plan rs_plan;
typedef struct rs_executor rs_executor;

/* ---- errors / hashing ---------------------------------------------------------------- */
const char* rs_last_error(void);
const char* rs_errc_name(int errc);
int rs_errc_count(void);
uint64_t rs_fnv1a64(const void* data, uint64_t n);
uint64_t rs_payload_seed(const char* path);
const char* rs_build_info(void);

/* ---- box algebra (host) ----------------------------------------------------------------- */
int rs_range_parse(const char* text, rs_range* out);
int rs_range_format(const rs_range* r, char* buf, uint64_t cap);
/* grid: npts[d] points for dim d, concatenated in pts */
int rs_grid_cells(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts, int cap,
                  rs_range* cells, int* n_cells);
int rs_grid_refine(int rank_a, const int32_t* npts_a, const uint64_t* pts_a, int rank_b, const int32_t* npts_b,
                   const uint64_t* pts_b, int32_t* npts_out, uint64_t* pts_out);
int rs_even_split(int rank, const uint64_t* shape, int dim, uint64_t ways, int32_t* npts_out, uint64_t* pts_out);
/* SplitGrid::cell / cell_index_of (split_grid.hpp:40-44, split_grid.cpp:88-117) */
int rs_grid_cell(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts, uint64_t index,
                 rs_range* out);
int rs_grid_cell_index_of(int rank, const uint64_t* shape, const int32_t* npts, const uint64_t* pts,
                          const rs_range* r, uint64_t* index);
/* Range::offset_by / valid_for (range.hpp:45-52, range.cpp:49-90) */
int rs_range_offset_by(const rs_range* r, const rs_range* outer, rs_range* out);
int rs_range_valid_for(const rs_range* r, int rank, const uint64_t* shape, int32_t* ok);
/* RangeSpec::parse + resolve (range.hpp:70-91, range.cpp:146-193): "[:,2:4]" -> box in shape */
int rs_rangespec_resolve(const char* spec, int rank, const uint64_t* shape, rs_range* out);
/* dtype_from_name (dtype.hpp:31, dtype.cpp:17-23) plus "bf16"/"BF16" */
int rs_dtype_from_name(const char* name, int32_t* code);

/* ---- device runtime -------------------------------------------------------------------- */
int rs_device_count(int* n);
/* A context drives `n_local` GPUs of a world of `world` GPUs: world_ids[i] runs on CUDA
 * device cuda_devices[i].  Single process: world = n_local, world_ids = 0..n-1. */
int rs_init(int world, int n_local, const int32_t* world_ids, const int32_t* cuda_devices, rs_context** out);
void rs_destroy(rs_context* ctx);
int rs_malloc(rs_context* ctx, int gpu, uint64_t bytes, void** out);
int rs_free(rs_context* ctx, int gpu, void* ptr);
int rs_host_alloc(uint64_t bytes, void** out); /* pinned host memory */
int rs_host_free(void* ptr);
int rs_memcpy_htod(rs_context* ctx, int gpu, void* dst, const void* src, uint64_t n);
int rs_memcpy_dtoh(rs_context* ctx, int gpu, void* dst, const void* src, uint64_t n);
int rs_memset(rs_context* ctx, int gpu, void* dst, int value, uint64_t n);
int rs_sync(rs_context* ctx, int gpu);
/* CUDA IPC for one-process-per-GPU worlds: 64-byte opaque handles */
int rs_ipc_get_handle(rs_context* ctx, int gpu, void* ptr, void* handle64);
int rs_ipc_open_handle(rs_context* ctx, int gpu, const void* handle64, void** out);
int rs_ipc_close_handle(rs_context* ctx, int gpu, void* ptr);

/* ---- tensor core on device (reference slice / merge semantics and error precedence) --- */
/* Stream events across processes (one process per GPU, SPEC.md:501's barriers on the device):
 * rs_ipc_event_create makes an interprocess event on `gpu` and writes its 64-byte handle;
 * another rank opens it with rs_ipc_event_open.  rs_event_record / rs_event_wait enqueue a
 * record / a wait on the GPU's context stream (a wait binds to the LAST record enqueued before
 * it — order them with a host barrier).  rs_timing_event_create + rs_event_elapsed time a span
 * on one GPU's stream (elapsed synchronizes on the second event).  `bench.py` under torchrun:
 * rank 0 records start + "go", every rank waits on "go" before its kernels and records "done",
 * rank 0 waits on every "done" and records the end: one common start, the last rank's end. */
typedef struct rs_event rs_event;
int rs_ipc_event_create(rs_context* ctx, int gpu, void* handle64, rs_event** out);
int rs_ipc_event_open(rs_context* ctx, int gpu, const void* handle64, rs_event** out);
int rs_timing_event_create(rs_context* ctx, int gpu, rs_event** out);
int rs_event_record(rs_context* ctx, int gpu, rs_event* ev);
int rs_event_wait(rs_context* ctx, int gpu, rs_event* ev);
int rs_event_elapsed(rs_event* start, rs_event* stop, float* ms);
void rs_event_destroy(rs_event* ev);

int rs_slice(rs_context* ctx, int gpu, const rs_tensor* t, const rs_range* r, void* out);
int rs_merge(rs_context* ctx, int gpu, int n_parts, const rs_range* ranges, const rs_tensor* parts, int rank,
             const uint64_t* target_shape, void* out);
/* SURVEY §8(b) rs_broadcast, without NCCL: `bytes` at `src` (device memory of world GPU `gpu`)
 * to every pointer of dsts[0..n_dst) (local or peer / IPC mappings) by one kernel on that GPU:
 * the source is read once per kMaxFan destinations and stored to each (TMA bulk fan-out tiles
 * when all pointers and `bytes` are 16-byte aligned).  DP replication as one push. */
int rs_broadcast(rs_context* ctx, int gpu, const void* src, int n_dst, void* const* dsts, uint64_t bytes,
                 rs_timing* timing);
/* The same on HOST buffers (t->data / parts[i].data / out are host pointers): the reference's
 * value-level slice / merge (tensor.hpp:40-47) — validated first, in the reference's order,
 * then staged through the context's GPU.  C++ callers get the reference's own value type
 * instead: reshard::Tensor, reshard::slice, reshard::merge (reshard/tensor.hpp). */
int rs_slice_host(rs_context* ctx, int gpu, const rs_tensor* t, const rs_range* r, void* out);
int rs_merge_host(rs_context* ctx, int gpu, int n_parts, const rs_range* ranges, const rs_tensor* parts, int rank,
                  const uint64_t* target_shape, void* out);

/* ---- collection description ------------------------------------------------------------- */
int rs_catalog_create(rs_catalog** out);
int rs_catalog_gpt(uint64_t hidden, uint64_t layers, uint64_t seq, uint64_t vocab, int state_kind, rs_catalog** out);
int rs_catalog_add(rs_catalog* c, const char* path, int dtype, int rank, const uint64_t* shape, int tp_dim, int layer);
int rs_catalog_size(const rs_catalog* c);
int rs_catalog_get(const rs_catalog* c, int i, char* path, int cap, int32_t* dtype, int32_t* rank, uint64_t* shape,
                   int32_t* tp_dim, int32_t* layer);
uint64_t rs_catalog_bytes(const rs_catalog* c);
void rs_catalog_destroy(rs_catalog* c);

int rs_build_strategy(const rs_catalog* c, int n_devices, const rs_device* devices, int tp, int pp, int dp,
                      rs_ptc** out);
void rs_ptc_destroy(rs_ptc* p);
/* test hooks mirroring the SPEC validate() examples */
int rs_ptc_set_alpha(rs_ptc* p, int partition, int n, const rs_device* devices);
int rs_ptc_set_sigma(rs_ptc* p, int tensor, int rank, const int32_t* npts, const uint64_t* pts);
int rs_validate(const rs_ptc* p, char* buf, uint64_t cap, int* n_violations);
int rs_hosted_subtensors(const rs_ptc* p, rs_device dev, int cap, int32_t* tensor, rs_range* cells, int* n);
int rs_ptc_devices(const rs_ptc* p, int cap, rs_device* out, int* n);
/* sigma cell `cell` of tensor `tensor` (lexicographic cell order, split_grid.cpp:62-86) */
int rs_ptc_cell(const rs_ptc* p, int tensor, int cell, rs_range* out);
int rs_ptc_cell_count(const rs_ptc* p, int tensor, int* n);

/* parallelization-configuration JSON: list by rank of model trees
 * whose leaves are {base, shape, range|null, dtype}.  devices may be NULL: rank r -> (0, r). */
int rs_parse_parallel_config(const char* json, int n_devices, const rs_device* devices, rs_ptc** out);
/* returns the bytes needed including NUL; writes at most cap bytes */
int64_t rs_serialize_parallel_config(const rs_ptc* p, char* buf, int64_t cap);

/* ---- planner ---------------------------------------------------------------------------- */
int rs_generate_plan(const rs_ptc* from, const rs_ptc* to, rs_plan** out);
int rs_recover(const rs_ptc* from, int n_failed, const rs_device* failed, const rs_ptc* to, rs_plan** out);
void rs_plan_destroy(rs_plan* p);
int rs_plan_get_stats(const rs_plan* p, rs_plan_stats* out);
int rs_plan_cost(const rs_plan* p, int cap, rs_device* devices, uint64_t* ingress, uint64_t* egress, int* n);
/* central-mode attribution: every Move routed through `central` */
int rs_plan_cost_central(const rs_plan* p, rs_device central, int cap, rs_device* devices, uint64_t* ingress,
                         uint64_t* egress, int* n);
/* returns the bytes needed including NUL; writes at most cap bytes */
int64_t rs_plan_text(const rs_plan* p, char* buf, int64_t cap);
int rs_choose_source(int n, const rs_device* candidates, const uint64_t* egress, rs_device dst, rs_device* out);

/* ---- executor (apply_plan data plane) --------------------------------------------------- */
/* src_gpu[i]: world GPU of from-device i; dst_gpu[j]: world GPU of to-device j */
int rs_executor_create(rs_context* ctx, const rs_plan* plan, const int32_t* src_gpu, const int32_t* dst_gpu,
                       uint64_t tile_bytes, rs_executor** out);
/* same, restricted to catalog tensors [t_begin, t_end): plans larger than the world's HBM
 * run as several windows (waves) over reused arenas */
int rs_executor_create_window(rs_context* ctx, const rs_plan* plan, const int32_t* src_gpu, const int32_t* dst_gpu,
                              uint64_t tile_bytes, uint32_t t_begin, uint32_t t_end, rs_executor** out);
/* apply_plan(plan, central) (the paper's §6.3 baseline): every moved
 * fragment goes source -> staging region on `central_gpu` -> destination, in two dependent
 * phases; same final state as distributed mode.  The staging region is the tail of the
 * central GPU's dst arena (rs_executor_arena_bytes includes it).  Every GPU of the world
 * must be local to the context. */
int rs_executor_create_central(rs_context* ctx, const rs_plan* plan, const int32_t* src_gpu, const int32_t* dst_gpu,
                               uint64_t tile_bytes, int central_gpu, rs_executor** out);
int rs_executor_staging_bytes(const rs_executor* e, uint64_t* bytes);
void rs_executor_destroy(rs_executor* e);
int rs_executor_arena_bytes(const rs_executor* e, int gpu, uint64_t* src_bytes, uint64_t* dst_bytes);
int rs_executor_bind(rs_executor* e, int gpu, void* src_arena, void* dst_arena);
int rs_executor_prepare(rs_executor* e);
int rs_executor_run(rs_executor* e);                     /* async launch on every local GPU */
int rs_executor_wait(rs_executor* e, int cap, rs_timing* out, int* n); /* per local GPU */
/* end to end on host buffers (single-GPU world): H2D src arena, copy kernel, D2H dst arena,
 * all on the GPU's stream and bracketed by CUDA events; arenas must be bound */
int rs_executor_run_host(rs_executor* e, int gpu, const void* host_src_arena, void* host_dst_arena, rs_timing* out);
/* The same with flags.  RS_HOST_SKIP_UNREAD: host -> device copies of only the source ranges
 * the copy tiles read (pipelined path); source state no tile reads (cells a reshard keeps in
 * place, e.g. the survivors' own cells in a recovery) stays in the host buffer and the device
 * src arena is not refreshed there.  rs_executor_host_upload_bytes: the bytes such a call copies
 * host -> device.  Unknown flag bits: InvalidArgument. */
#define RS_HOST_SKIP_UNREAD 1u
int rs_executor_run_host_flags(rs_executor* e, int gpu, const void* host_src_arena, void* host_dst_arena,
                               unsigned flags, rs_timing* out);
int rs_executor_host_upload_bytes(rs_executor* e, int gpu, unsigned flags, uint64_t* bytes);
/* multi-process end-to-end step in phases separated by the caller's cross-rank barriers:
 * 0 = start mark + H2D of the GPU's src arena (host_buf = src), 1 = kernels (host_buf
 * unused), 2 = D2H of its dst arena (host_buf = dst) + stop mark; each phase returns after
 * its stream work completes.  rs_executor_host_elapsed: event time mark to mark. */
int rs_executor_host_phase(rs_executor* e, int gpu, int phase, void* host_buf);
int rs_executor_host_elapsed(rs_executor* e, int gpu, float* ms);
/* World time of the last rs_executor_wait: from one common start mark (recorded on the first
 * local GPU, waited on by every other local GPU before its kernels) to the end of the last local
 * GPU's kernels, peer pushes included (single-process multi-GPU worlds; = the GPU's own time
 * for one local GPU).  Replaces SPEC.md:501's "timestamps across all participating workers". */
int rs_executor_world_ms(const rs_executor* e, float* ms);
/* End to end through host buffers over every local GPU of a single-process world, from one
 * common start to the last D2H (*ms).  Default: pipelined rounds — every GPU's tile lists cut
 * into chunks; round k uploads the source ranges chunk k first reads, runs chunk k on every GPU,
 * and once chunk k is done everywhere moves down each dst-arena prefix no later chunk writes,
 * so H2D, pushes and D2H overlap on every link.  RESHARD_WORLD_PIPELINE=0 (or a world with
 * non-local GPUs): H2D of every src arena, each GPU's kernels once its own src arena landed,
 * world barrier, D2H of every dst arena.  host_src / host_dst: n = world
 * entries, indexed by world GPU (entries of non-local GPUs are ignored). */
int rs_executor_run_host_world(rs_executor* e, int n, const void* const* host_src, void* const* host_dst, float* ms);
/* ExecutionReport verification digests: per base tensor of the executor's
 * window, FNV-1a-64 (hash.hpp:13-42) of the tensor reassembled from one replica of each cell of
 * side 0 (source layout) or 1 (destination layout), read back from the local GPUs (off the
 * clock).  replica: which DP copy of a cell (0 = the first in layout order, -1 = the last; the
 * nearest existing one when a cell has fewer).  ok[i] = 0 when a cell of tensor[i] is not held
 * by a local GPU.  *n = entries. */
int rs_executor_digests(rs_executor* e, int side, int replica, int cap, int32_t* tensor, uint64_t* fnv, int32_t* ok,
                        int* n);
int rs_executor_fill_sources(rs_executor* e);
int rs_executor_verify(rs_executor* e, uint64_t* mismatched_bytes);
/* bindings: src cells in (from-device, tensor, cell) order; dst cells in plan order */
int rs_executor_src_cells(const rs_executor* e, int cap, rs_cell_binding* out, int* n);
int rs_executor_dst_cells(const rs_executor* e, int cap, rs_cell_binding* out, int32_t* dst_device, int32_t* tensor,
                          int32_t* cell, int* n);
int rs_executor_tiles(const rs_executor* e, int gpu, uint64_t* tiles, uint64_t* bytes);
int rs_executor_read_bytes(const rs_executor* e, int gpu, uint64_t* bytes);
/* bytes GPU `gpu`'s tiles write into each world GPU (bytes[w], n >= world): the egress row
 * of the fragment all-to-all; bytes[gpu] are its local HBM writes */
int rs_executor_bytes_to(const rs_executor* e, int gpu, int n, uint64_t* bytes);

/* ---- PTX1 container and checkpoints (ptx_io.hpp:10-20) ------------
 * PTX1 defines dtype codes 0..3 only: BF16 (4) payloads are WRITTEN WITH THE F16 CODE (1), same
 * width, so reference readers accept the files; decoding such a file yields F16.  A checkpoint
 * load takes the real dtype from the executor's layout, not from the file.
 * Checkpoint files: <dir>/<rank>/<tensor path>.ptx, or <tensor path>.c<cell>.ptx when the rank
 * hosts several cells of that tensor.  Tensor paths must be relative without '..'
 * (InvalidArgument).  A failed write or close is IoError. */
int rs_ptx_encoded_size(int dtype, int rank, const uint64_t* shape, uint64_t* bytes);
int rs_ptx_encode_header(int dtype, int rank, const uint64_t* shape, uint8_t* out, uint64_t cap, uint64_t* written);
/* validates a whole PTX1 buffer (header + payload) */
int rs_ptx_decode_header(const uint8_t* bytes, uint64_t n, int32_t* dtype, int32_t* rank, uint64_t* shape,
                         uint64_t* header_bytes);
/* side 0: the plan's source layout (src arena); side 1: its destination layout */
int rs_checkpoint_save(rs_executor* e, int side, const char* dir, uint64_t* files, uint64_t* bytes, double* seconds);
int rs_checkpoint_load(rs_executor* e, const char* dir, uint64_t* files, uint64_t* bytes, double* seconds);

/* ---- dataset index repartitioning ------------------------------------- */
/* shuffle_epoch: Fisher-Yates (i = N-1 .. 1, j = next_below(i+1)), splitmix64 seeded seed^epoch */
int rs_shuffle_epoch(uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm_host);
int rs_repartition_count(uint64_t n, uint64_t global_batch, uint64_t at_step, uint64_t new_dp, uint64_t rank,
                         uint64_t* count);
int rs_repartition_position(uint64_t n, uint64_t global_batch, uint64_t at_step, uint64_t new_dp, uint64_t rank,
                            uint64_t k, uint64_t* pos);
/* locate_sample on host arrays: out = {file, offset, length, locator class} */
int rs_locate_sample(uint64_t n, uint64_t global_batch, uint64_t at_step, uint64_t new_dp, uint64_t rank,
                     uint64_t k, const uint64_t* perm, const uint64_t* samples, const uint8_t* file_class,
                     uint64_t* out4);

typedef struct rs_dataset_index {  /* device pointers */
  const uint64_t* perm;          /* N: epoch permutation */
  const uint64_t* samples;       /* N x {file, offset, length} */
  const uint8_t* file_class;     /* per file: 0 local, 1 peer, 2 remote for the calling rank */
  uint64_t n;
  uint64_t entry_bytes;          /* 0 or 24: packed records as the reference stores them;
                                    32: padded device layout from rs_dataset_index_pad */
} rs_dataset_index;

typedef struct rs_partition_out {  /* device pointers, capacity = the rank's count */
  uint64_t* pos;                 /* global positions */
  uint64_t* ent;                 /* 3 x u64 per sample */
  uint64_t* boff;                /* exclusive prefix sum of lengths */
  uint32_t* queue[3];            /* sample indices k per locator class, increasing */
  uint64_t* qcount;              /* 3 counts, written by the kernel */
} rs_partition_out;

typedef struct rs_partition_host {  /* host pointers (pinned for full PCIe rate) */
  uint64_t* pos;
  uint64_t* ent;
  uint64_t* boff;
  uint32_t* queue[3];            /* receives exactly qcount[c] entries */
  uint64_t* qcount;
} rs_partition_host;

/* K8: shuffle_epoch on the GPU, bit-identical to rs_shuffle_epoch (deterministic
 * reservations, kept in the high words of perm_dev while it runs); n < 2^32; perm_dev: n x u64
 * device buffer; scratch: rs_shuffle_scratch_bytes(n) (the carried-iteration lists, 16 B per
 * window entry: max(n/20, 64 Ki) entries).  Synchronous; timing->tiles = rounds. */
int rs_shuffle_scratch_bytes(uint64_t n, uint64_t* bytes);
int rs_shuffle_epoch_device(rs_context* ctx, int gpu, uint64_t n, uint64_t seed, uint64_t epoch, uint64_t* perm_dev,
                            void* scratch, rs_timing* timing);

/* Device layout of the index (no reference counterpart; the index is static across epochs
 * and DP changes, so this runs once per index load): packed 24-byte records -> padded
 * 32-byte records (padded: n x 32 bytes, 16-byte aligned).  rs_repartition's outputs are
 * identical for either layout; the padded one never straddles a DRAM line. */
int rs_dataset_index_pad(rs_context* ctx, int gpu, const uint64_t* packed_dev, uint64_t* padded_dev, uint64_t n,
                         rs_timing* timing);
/* Host-buffer path (the SPEC's dataset module works on host-resident indexes):
 * upload perm (8n B) and the packed records (24n B) into perm_dev / samples_dev on the GPU's
 * stream; with padded_dev non-null also rewrite them padded (rs_dataset_index_pad).  timing->ms:
 * event time of the upload. */
int rs_dataset_index_upload(rs_context* ctx, int gpu, const uint64_t* host_perm, const uint64_t* host_samples,
                            uint64_t n, uint64_t* perm_dev, uint64_t* samples_dev, uint64_t* padded_dev,
                            rs_timing* timing);
int rs_repartition_scratch_bytes(uint64_t count, uint64_t* bytes);
/* K5: gather pass + tile scan + finalize for one rank (three launches, timed with events;
 * timing->main_ms = the gather pass alone).  Replaces the SPEC's per-rank repartition +
 * locate_sample loops. */
int rs_repartition(rs_context* ctx, int gpu, const rs_dataset_index* idx, uint64_t global_batch, uint64_t at_step,
                   uint64_t new_dp, uint64_t rank, const rs_partition_out* out, void* scratch, rs_timing* timing);
/* Several ranks' K5 on one GPU (a GPU hosting several new DP ranks).  Default: every rank in
 * ONE launch per pass (gather, tile scan, finalize; a block finds its rank from a rank table),
 * so there is no launch tail between ranks (the default gather variant; RESHARD_K5 /
 * RESHARD_K5_LOAD A/B variants take the unfused schedule).  RESHARD_K5_FUSE=0: the gather passes back to back
 * on a high-priority stream, each rank's tile scan + finalize on a low-priority second stream.
 * idx->file_class is ignored: each job names its own (locator classes differ per rank).
 * total->ms: batch start to the last finalize (events); total->main_ms: the gather pass(es);
 * per_job (nullable, n entries): tiles and algorithmic bytes, and with RESHARD_K5_FUSE=0 each
 * rank's gather-pass time in ms / main_ms (0 when fused: one launch serves every rank).  Same
 * outputs as n rs_repartition calls. */
typedef struct rs_repartition_job {
  uint64_t at_step, new_dp, rank;
  const uint8_t* file_class;     /* device, per file: 0 local, 1 peer, 2 remote for this rank */
  rs_partition_out out;
  void* scratch;                 /* rs_repartition_scratch_bytes(count), device */
} rs_repartition_job;
int rs_repartition_batch(rs_context* ctx, int gpu, const rs_dataset_index* idx, uint64_t global_batch,
                         const rs_repartition_job* jobs, int n, rs_timing* per_job, rs_timing* total);
/* rs_repartition, then the rank's outputs back to host buffers on the same stream (count
 * entries of pos / ent / boff, qcount[c] entries of queue c).  timing->ms: kernels + D2H,
 * timing->main_ms: the gather pass, timing->bytes: D2H bytes. */
int rs_repartition_to_host(rs_context* ctx, int gpu, const rs_dataset_index* idx, uint64_t global_batch,
                           uint64_t at_step, uint64_t new_dp, uint64_t rank, const rs_partition_out* out,
                           void* scratch, const rs_partition_host* host, rs_timing* timing);
/* Diagnostic (no reference counterpart): best-of-`reps` device time of K5's perm + entry
 * gathers for this rank plus all 44 output bytes per sample written coalesced, no scan
 * (env RESHARD_PROBE=read: nothing written) — the floor bench.py reports K5 against.
 * idx->file_class is not read. */
int rs_repartition_gather_probe(rs_context* ctx, int gpu, const rs_dataset_index* idx, uint64_t global_batch,
                                uint64_t at_step, uint64_t new_dp, uint64_t rank, int reps, rs_timing* timing);

#ifdef __cplusplus
}
#endif

#endif /* RESHARD_B200_H */
