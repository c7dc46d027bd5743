/*
 * pgx.h — C ABI of the B200-native per-layer gradient exchange (libpgx.so).
 *
 * Drop-in boundary for the hot path of arXiv 1706.00095 as restated by the
 * reference package `pipesgd` (/root/reference/pkg/src/pipesgd).  Every entry
 * point below names the reference interface it replaces (file:line relative to
 * that directory).  Plain pointers, sizes and integer status codes only; a
 * `cudaStream_t` is passed as `void*` (NULL = the legacy default stream).
 *
 * Status codes map one-to-one onto the reference's exception taxonomy
 * (errors.py:8-50); `pgx_last_error()` returns the message of the most recent
 * failure on the calling thread.
 */
#ifndef PGX_H_
#define PGX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGX_ABI_VERSION 3
#define PGX_IPC_HANDLE_BYTES 64
#define PGX_CONTROL_SEGMENT 15 /* transport/base.py:21 */
#define PGX_MAX_RANKS 8
#define PGX_MAX_PIECES 4

enum pgx_status {
  PGX_OK = 0,
  PGX_E_SHAPE = 1,     /* ShapeError      errors.py:8  */
  PGX_E_INPUT = 2,     /* InputError      errors.py:12 */
  PGX_E_CONFIG = 3,    /* ConfigError     errors.py:16 */
  PGX_E_RANGE = 4,     /* RangeError      errors.py:20 */
  PGX_E_ROUTING = 5,   /* RoutingError    errors.py:24 */
  PGX_E_TREE = 6,      /* TreeError       errors.py:28 */
  PGX_E_TRANSPORT = 7, /* TransportError  errors.py:32 */
  PGX_E_PROTOCOL = 8,  /* ProtocolError   errors.py:36 */
  PGX_E_TIMEOUT = 9,   /* TransportError (bounded device/host wait expired) */
  PGX_E_CUDA = 10,     /* TransportError (CUDA runtime failure) */
  PGX_E_FORMAT = 11    /* FormatError     errors.py:49 */
};

typedef struct pgx_world pgx_world;
typedef struct pgx_xchg pgx_xchg;

int pgx_abi_version(void);
const char* pgx_last_error(void);

/* ------------------------------------------------------------------ world
 * One per rank (one process per GPU, or several ranks in one process on one
 * GPU for host-stepped tests).  Replaces TransportBase.__init__
 * (transport/base.py:173-183) + InprocWorld (transport/inproc.py:62-127). */
int pgx_world_create(int rank, int world_size, int device, pgx_world** out);
int pgx_world_destroy(pgx_world* w);
/* Per-rank device status word (0 = ok); bounded device waits write
 * PGX_E_TIMEOUT here.  Host-mapped, readable without a sync. */
int pgx_world_status(pgx_world* w, uint32_t* status_out);
int pgx_world_clear_status(pgx_world* w);
int pgx_world_set_timeout(pgx_world* w, double seconds);

/* -------------------------------------------------------------- segments
 * segment_create (base.py:185-194): id < 65536, != 15 unless internal,
 * size >= 1, notification_count >= 1; duplicate id -> PGX_E_CONFIG.
 * Memory is cudaMalloc'ed, zeroed, IPC-exportable: [data | pad | u32 flags]. */
int pgx_segment_create(pgx_world* w, uint32_t seg_id, uint64_t size, uint32_t notif_count,
                       void** data_out, uint32_t** flags_out);
/* Any rank's view of a segment (own or attached peer).  segment() base.py:196 */
int pgx_segment_info(pgx_world* w, int rank, uint32_t seg_id, void** data_out,
                     uint32_t** flags_out, uint64_t* size_out, uint32_t* count_out);
/* Export / attach: the rendezvous that makes peer segments one-sided
 * writable.  Handles travel between processes as opaque 64-byte blobs. */
int pgx_segment_export(pgx_world* w, uint32_t seg_id, void* handle_out);
int pgx_segment_attach_ipc(pgx_world* w, int peer, uint32_t seg_id, const void* handle,
                           uint64_t size, uint32_t notif_count);
int pgx_segment_attach_local(pgx_world* w, int peer, uint32_t seg_id, void* data,
                             uint32_t* flags, uint64_t size, uint32_t notif_count);
/* Several ranks on distinct GPUs inside ONE process (host-stepped multi-GPU tests and
 * per-phase microbenchmarks): let `device` address `peer`'s memory directly. */
int pgx_enable_peer_access(int device, int peer);

/* ------------------------------------------------------------ data plane
 * write_notify (inproc.py:134-142, base.py:217-225 validation): copy `size`
 * bytes from the local segment into the remote rank's segment with device
 * stores (NVLink peer stores when remote), then raise notification `nid` to
 * `value` with a system-scope release.  Non-blocking: enqueued on `stream`.
 * value 0 -> PGX_E_PROTOCOL; bad ranges -> PGX_E_RANGE; bad rank ->
 * PGX_E_ROUTING. */
int pgx_write_notify(pgx_world* w, uint32_t local_seg, uint64_t local_off, int rank,
                     uint32_t remote_seg, uint64_t remote_off, uint64_t size, uint32_t nid,
                     uint32_t value, void* stream);
/* The chunked transfer of RankBase._send (engine/runtime.py:185-224) in one
 * launch: ceil(size/chunk_bytes) chunks, chunk j raising id
 * chunk_notification_id(base_id, j, n) (engine/layout.py:130-139). */
int pgx_write_notify_chunked(pgx_world* w, uint32_t local_seg, uint64_t local_off, int rank,
                             uint32_t remote_seg, uint64_t remote_off, uint64_t size,
                             uint64_t chunk_bytes, uint32_t base_id, uint32_t value,
                             void* stream);
/* notify_poll (base.py:110-119 / 203): non-consuming; writes the fired
 * (id, value) pairs in [first, first+count) in ascending id order. */
int pgx_notify_poll(pgx_world* w, uint32_t seg_id, uint32_t first, uint32_t count,
                    uint32_t* ids_out, uint32_t* values_out, uint32_t capacity,
                    uint32_t* n_out);
/* notify_reset (base.py:121-126 / 206): atomic consume-once; old value or 0. */
int pgx_notify_reset(pgx_world* w, uint32_t seg_id, uint32_t nid, uint32_t* old_out);

/* Tickets (base.py:58-91): a CUDA event recorded after the write. */
int pgx_ticket_record(void* stream, void** ticket_out);
int pgx_ticket_query(void* ticket); /* 1 = done, 0 = pending, <0 error */
int pgx_ticket_wait(void* ticket, double timeout_s); /* ticket_wait_all base.py:210 */
int pgx_ticket_release(void* ticket);

/* Device flag barrier over CONTROL_SEGMENT (tcp.py:229-269 analog). Only for
 * ranks on distinct GPUs; host-stepped single-GPU worlds barrier on the host. */
int pgx_barrier(pgx_world* w, void* stream, double timeout_s);
/* The same device barrier enqueued on `stream` without waiting for it on the host (ranks
 * leave it within one flag round trip of each other: used to align timed regions). */
int pgx_barrier_async(pgx_world* w, void* stream, double timeout_s);

/* ------------------------------------------------------------ arithmetic
 * buffer_axpy (buffers.py:69-74): y := y + (alpha*x), two roundings. */
int pgx_axpy_f64(double alpha, const double* x, double* y, uint64_t n, void* stream);
int pgx_axpy_f32(float alpha, const float* x, float* y, uint64_t n, void* stream);
/* master_update (engine/sgd.py:27-33): out = w - eps*g in float64 (two
 * roundings, no FMA).  The f32 entry takes fp32 w/g, promotes like numpy and
 * stores the float64 result rounded to fp32 ("ref32"). */
int pgx_master_update_f64(const double* w, const double* g, double eps, double* out,
                          uint64_t n, void* stream);
int pgx_master_update_f32(const float* w, const float* g, double eps, float* out,
                          uint64_t n, void* stream);
/* tree_reduce (engine/sgd.py:53-69): out = root sum of `world` partials
 * folded in binomial-tree order (children ascending).  `partials` is a HOST
 * array of `world` device pointers.  f64: reference-native; f32: ref32. */
int pgx_tree_reduce_f64(const double* const* partials, int world, double* out, uint64_t n,
                        void* stream);
int pgx_tree_reduce_f32(const float* const* partials, int world, float* out, uint64_t n,
                        void* stream);

/* Fused fold + update modes. */
enum pgx_mode {
  PGX_MODE_REF64 = 0,  /* f64 storage, bit-exact with the reference engine      */
  PGX_MODE_REF32 = 1,  /* f32 storage, reference ops applied to fp32 arrays      */
  PGX_MODE_FAST32 = 2, /* f32: g*scale + wd*w, v = mu*v + lr*g, w -= v           */
  PGX_MODE_SUM32 = 3   /* f32, update off: w = scale * (tree-order sum) — an all-reduce
                          (average) with the same fold order; the sweep's NCCL peer */
};
/* Master-side fused _advance_folds + _apply_update (pipelined.py:103-108,
 * 158-188): tree-order fold of `world` partials, then the update in place on
 * w (and v for FAST32).  `partials` is a HOST array of device pointers;
 * element type f64 for REF64, f32 otherwise. */
int pgx_fold_update(int mode, const void* const* partials, int world, void* w, float* v,
                    uint64_t n, double eps, float scale, float momentum, float weight_decay,
                    void* stream);
/* ------------------------------------------------------------------ checkpoints
 * PSGD1 model checkpoints (engine/checkpoint.py:1-71): "PSGD1", then per layer
 * u32 index, u64 count, count x f64 (little-endian).  Replaces serialize_model
 * (:29-39) and load_model_bytes (:42-63): the image is built / read by one device
 * kernel from / into the layers (fp32 layers are promoted exactly / rounded to
 * nearest); header validation is host code with the reference's FormatError
 * messages. */
#define PGX_CKPT_MAX_LAYERS 512  /* layers whose table travels as the kernel parameter; more
                                    layers use a stream-ordered device copy (no format limit) */
/* image bytes = 5 + sum(12 + 8*count) */
int pgx_ckpt_image_bytes(const uint64_t* counts, int num_layers, uint64_t* bytes_out);
/* Host: walk and validate a PSGD1 blob (load_model_bytes, checkpoint.py:42-63);
 * counts_out may be NULL (count only).  PGX_E_FORMAT with the reference messages. */
int pgx_ckpt_parse(const void* blob, uint64_t bytes, uint64_t* counts_out, int capacity, int* num_layers_out);
/* Device: layers (elem_size 4 or 8) -> image (16-byte aligned, capacity >= bytes
 * rounded up to 16; the pad bytes are zero). */
int pgx_ckpt_pack(const void* const* layers, const uint64_t* counts, int num_layers, int elem_size, void* image,
                  uint64_t capacity, void* stream);
/* Device: image (8-byte aligned, capacity >= bytes rounded up to 8, plus 8) -> layers. */
int pgx_ckpt_unpack(const void* image, uint64_t capacity, const uint64_t* counts, int num_layers, int elem_size,
                    void* const* layers, void* stream);

/* seeded_fill (buffers.py:54-66) on the device, bit-identical to numpy. */
int pgx_seeded_fill_f64(uint64_t seed, double scale, double* out, uint64_t n, void* stream);
int pgx_seeded_fill_f32(uint64_t seed, double scale, float* out, uint64_t n, void* stream);

/* ------------------------------------------------- device-driven exchange
 * The fast path: per-layer pipelined gradient exchange with device-side
 * acquire waits (no host polling, no barrier).  One object per rank; its
 * receive segments live in the rank's world and are attached like any other.
 *
 * Variants (per layer):  TREE    = the paper's binomial reduce to rank 0,
 *                                  master update, broadcast down the same edges;
 *                        TWOSHOT = one-sided reduce-scatter to shard owners,
 *                                  owner fold (same tree order) + fused update,
 *                                  one-sided all-gather into peers' weights;
 *                        ONESHOT = every rank pushes its whole gradient to every
 *                                  peer and updates its own copy (small layers).
 * TREE, TWOSHOT(_CE/_CEP) and ONESHOT(_LL) are bit-identical to the reference fold order;
 * NVLS reduces in the switch (fast32, tolerance parity). */
enum pgx_variant {
  PGX_VARIANT_TREE = 0,       /* paper: binomial reduce + master update + broadcast     */
  PGX_VARIANT_TWOSHOT = 1,    /* SM peer stores: reduce-scatter, owner update, gather   */
  PGX_VARIANT_TWOSHOT_CE = 2, /* same schedule, shards moved by the copy engines        */
  PGX_VARIANT_NVLS = 3,       /* NVLink SHARP: in-switch reduce (multimem.ld_reduce) +
                                 multicast weight store; fast32 only, tolerance parity  */
  PGX_VARIANT_ONESHOT = 4,    /* small layers: everyone pushes everything once, every
                                 rank folds (same order) and updates its own copy       */
  PGX_VARIANT_TWOSHOT_CEP = 5,/* reduce-scatter by the copy engines, then the SM owner
                                 kernel (fold + update + all-gather peer stores) on a
                                 capped grid: no per-part copy/event chain            */
  PGX_VARIANT_ONESHOT_LL = 6,  /* small fp32 layers, fence-free: ONESHOT with every value
                                 carried as an 8-byte {value, epoch} word (2x bytes)  */
  PGX_VARIANT_ONESHOT_L128 = 7,/* fp32 ONESHOT over 128-byte lines: 30 values + an 8-byte
                                 epoch flag per line, fence-free (128/120 bytes); needs
                                 PGX_XF_ALLOW_L128 (the 128-byte write atomicity NCCL's
                                 LL128 protocol also rests on; stress-tested, r5c)     */
  PGX_VARIANT_TWOSHOT_BULK = 8,/* TWOSHOT with every NVLink byte moved by TMA bulk copies
                                 (cp.async.bulk through a shared-memory ring, one thread
                                 per CTA) on a capped grid, one system fence + flag per
                                 ~1 MB slab: the large-layer variant                     */
  PGX_VARIANT_TWOSHOT_L128 = 9 /* fp32 TWOSHOT over the ONESHOT_L128 line format: shards
                                 pushed as 128-byte lines to their owner, updated lines
                                 gathered into every peer's staging area and installed
                                 there; fence-free (mid-size layers); PGX_XF_ALLOW_L128  */
};

/* pgx_xchg_config.flags (ABI 3: these were process-environment knobs before) */
enum pgx_xchg_flag {
  PGX_XF_CE_RS_PARTS = 1,          /* TWOSHOT_CE: part-major push with per-part signals     */
  PGX_XF_TMA = 2,                  /* TWOSHOT: push + all-gather as TMA bulk copies          */
  PGX_XF_ONESHOT_SMALL_CHUNKS = 4, /* ONESHOT: ~one chunk per SM (measured slower, r3v)      */
  PGX_XF_AUTO_CHUNK_TREE = 8,      /* TREE: size-scaled chunks (measured slower, r3r)        */
  PGX_XF_NO_AUTO_CHUNK_NVLS = 16,  /* NVLS: keep chunk_elems instead of size-scaled chunks   */
  PGX_XF_ALLOW_L128 = 32,          /* permit ONESHOT_L128 / TWOSHOT_L128 layers (sm_100 only) */
  PGX_XF_BULK_LEAN = 64,           /* TWOSHOT_BULK: 256 threads + 64 KB ring per CTA (shares
                                      SMs with the backward) instead of 512 + 224 KB        */
  PGX_XF_BULK_CE_RS = 128,         /* TWOSHOT_BULK: reduce-scatter by the copy engines in
                                      part-major copies (per-part chunk signals); the kernel
                                      runs the owner slabs only (fold + update + TMA gather) */
  PGX_XF_CE_TMA_OWNER = 256,       /* TWOSHOT_CE: owner fold fed by TMA bulk loads on a capped
                                      grid (layer_max_ctas, default 32) instead of the LSU
                                      fold on every SM                                      */
  PGX_XF_LEAN_CAPPED = 512         /* ONESHOT_LL / TWOSHOT_L128 layers with a layer_max_ctas
                                      cap launch 128-thread CTAs (fewer SM slots held while
                                      they poll for their peers, next to the backward)      */
};

typedef struct pgx_xchg_config {
  int num_layers;
  const uint64_t* layer_elems;   /* S_l, elements per layer ([W row-major][b]) */
  const int* variant;            /* per layer pgx_variant */
  int mode;                      /* pgx_mode (REF64 uses double elements) */
  uint64_t chunk_elems;          /* notification granularity, multiple of 4; with N > 1
                                    the two-shot variants double it up to 65536 while a
                                    shard still has >= 128 chunks (fewer system fences);
                                    with N = 1 the two-shot (the fused update alone) caps
                                    it at 4096 (shorter last wave)                      */
  double lr;                     /* epsilon / learning rate */
  float scale, momentum, weight_decay;
  uint32_t seg_base;             /* segment ids seg_base (weights + arrival flags) and
                                    seg_base+1 (receive slots + their flags) */
  int max_ctas;                  /* CTAs per exchange launch (0 = auto) */
  const uint64_t* layer_chunk_elems; /* optional per-layer chunk_elems (NULL or 0 = chunk_elems) */
  const int* layer_max_ctas;     /* optional per-layer CTA cap (NULL or 0 = max_ctas) */
  /* ABI 3 (0 = the default everywhere) */
  int ce_parts;                  /* TWOSHOT_CE owner pipelining depth 1..8 (0 = 4)       */
  int ce_rs_streams;             /* TWOSHOT_CE reduce-scatter copy streams 1..2 (0 = 1)  */
  uint32_t flags;                /* pgx_xchg_flag bits                                    */
} pgx_xchg_config;

int pgx_xchg_create(pgx_world* w, const pgx_xchg_config* cfg, pgx_xchg** out);
int pgx_xchg_destroy(pgx_xchg* x);
/* Flat model buffer of this rank (layer l at element offset model_offset[l]),
 * IPC-exported as segment seg_base; frameworks alias parameters into it. */
int pgx_xchg_model(pgx_xchg* x, void** model_out, uint64_t* offsets_out);
/* After every rank attached every peer's segments in its world. */
int pgx_xchg_connect(pgx_xchg* x);
/* Launch layer l's exchange for iteration k on `stream`.  The layer gradient
 * is given as up to PGX_MAX_PIECES device pieces covering [0, S_l) in order
 * (e.g. dW then db).  Never blocks the host.  `phases` selects the parts to
 * launch (PGX_PHASE_ALL in production; host-stepped single-GPU tests launch
 * the phases of all ranks in dependency order so no kernel ever spins on a
 * kernel that has not been launched). */
enum pgx_phase {
  PGX_PHASE_PUSH = 1,  /* TWOSHOT reduce-scatter stores / TREE up pass           */
  PGX_PHASE_OWNER = 2, /* TWOSHOT owner fold + update + all-gather stores         */
  PGX_PHASE_DOWN = 4,  /* TREE broadcast forwarding on inner ranks                */
  PGX_PHASE_ALL = 7
};
int pgx_xchg_layer(pgx_xchg* x, int layer, uint32_t iteration, const void* const* pieces,
                   const uint64_t* piece_elems, int num_pieces, int phases, void* stream);
/* Make `stream` wait until layer l's updated weights of iteration k are in
 * this rank's model buffer (forward-pre-hook gate, replaces
 * finalize_iteration's global drain, pipelined.py:60-80). */
int pgx_xchg_gate(pgx_xchg* x, int layer, uint32_t iteration, void* stream);
/* Graph mode: take the iteration from a device counter instead of the host
 * argument, so a captured step (CUDA graph) replays with fresh epochs.
 * `current` = the last iteration already launched (0xFFFFFFFF = none); each
 * pgx_xchg_tick (captured at the start of a step) advances it by one.  In this
 * mode pgx_xchg_gate's `iteration` is relative: 0xFFFFFFFF = the previous
 * iteration (forward-pre-hook gate), 0 = the current one (end-of-step drain). */
int pgx_xchg_device_iteration(pgx_xchg* x, int enable, uint32_t current);
int pgx_xchg_tick(pgx_xchg* x, void* stream);
/* Internal streams (0 = tree down pass, 1 = CE reduce-scatter, 2 = CE owner side,
 * 3 = CE all-gather, 4 = CE second push stream). */
int pgx_xchg_stream(pgx_xchg* x, int which, void** stream_out);
/* Replace the internal streams by caller-owned ones (e.g. framework streams whose
 * lifetime the framework's allocator tracks); the library will not destroy them.
 * Order: tree down pass, CE push, CE owner, CE all-gather, CE second push. */
#define PGX_XCHG_STREAMS 5
int pgx_xchg_set_streams(pgx_xchg* x, void* const* streams, int n);
/* Make `stream` wait until layer l's local exchange work (own shard, side
 * streams) finished — joins every internal stream back (graph capture). */
int pgx_xchg_join(pgx_xchg* x, int layer, void* stream);
/* Kernels this exchange object has launched so far (exchange + gate kernels). */
int pgx_xchg_launch_count(pgx_xchg* x, uint64_t* count_out);
/* NVLS setup, collective over the ranks (after pgx_xchg_create, before use):
 * rank 0 creates the multicast object and exports it as a POSIX fd (others get -1);
 * the caller passes that fd to every other rank (SCM_RIGHTS); every rank imports it
 * and adds its GPU; after ALL ranks added, every rank binds its local memory.  The
 * weights then live in the multicast-backed buffer (re-query pgx_xchg_model). */
int pgx_xchg_nvls_export(pgx_xchg* x, int* fd_out);
int pgx_xchg_nvls_import(pgx_xchg* x, int fd);
int pgx_xchg_nvls_bind(pgx_xchg* x);
/* Whole-model gate: one launch waiting for every layer's arrivals of `iteration`
 * (same relative convention as pgx_xchg_gate in device-iteration mode). */
int pgx_xchg_gate_all(pgx_xchg* x, uint32_t iteration, void* stream);
/* Per-layer launch statistics for the roofline (bytes moved per launch). */
int pgx_xchg_layer_bytes(pgx_xchg* x, int layer, uint64_t* nvlink_out_bytes,
                         uint64_t* hbm_bytes);
/* The plan a layer runs with: effective chunk elements (notification granularity) and
 * CTAs of its exchange kernel launch. */
int pgx_xchg_layer_plan(pgx_xchg* x, int layer, uint64_t* chunk_elems_out, int* ctas_out);
/* TWOSHOT_CE: how many pipelined parts this rank's owner shard of `layer` is split into
 * (1 for every other variant). */
int pgx_xchg_layer_parts(pgx_xchg* x, int layer, int* parts_out);
/* Debug timeline: when `device_buffer` (u64 [items][8]) is non-NULL, instrumented kernels
 * (ONESHOT) stamp each work item's claim / mid / end globaltimer ns and SM id into it.
 * NULL turns it off (the default: one predicated-off branch per item). */
int pgx_xchg_set_trace(pgx_xchg* x, void* device_buffer);

/* Step graphs (no reference counterpart: the captured training step of bench.py).
 * Instantiate a captured cudaGraph_t with the capture streams' priorities kept on its
 * kernel nodes (cudaGraphInstantiateFlagUseNodePriority: the exchange stream's high
 * priority survives into the replays), launch it on `stream`, destroy the executable. */
int pgx_graph_instantiate_prio(void* graph, void** exec_out);
int pgx_graph_launch(void* exec, void* stream);
int pgx_graph_exec_destroy(void* exec);

#ifdef __cplusplus
}
#endif

#endif /* PGX_H_ */
