/*
 * dagrt.h -- C ABI of the run-time DAG scheduler (libdagrt.so).
 *
 * B200-native re-design of the scheduler of arXiv 2012.09646, "DAG-based
 * Scheduling with Resource Sharing for Multi-task Applications in a Polyglot
 * GPU Runtime".  Citations "Lnnn" are lines of the paper text.
 *
 * The user registers device arrays, declares kernels whose pointer arguments
 * are const (read-only) or mutable, launches kernels and touches arrays from
 * the host, writing host code "as if it were run sequentially, with no
 * explicit mention of synchronization points or streams" (L528-530).  The
 * library infers the computation DAG at run time from the read/write argument
 * sets (L386-430, L490-491), assigns CUDA streams (L570-582, L647-654), wires
 * cudaEvent / cudaStreamWaitEvent edges (L546-553), keeps the host-sync
 * frontier of active computations (L553-558) and overlaps host<->device
 * transfers with compute on side streams (L356-366, L662-664).
 *
 * Conventions for every call:
 *  - returns dagrt_status: 0 = DAGRT_OK, < 0 = error (enum below); no C++
 *    exception or longjmp ever crosses this boundary;
 *  - on error, dagrt_last_error(ctx) returns a NUL-terminated message owned by
 *    the context (valid until the next call on it);
 *  - a CUDA error makes the context sticky-failed: every later call returns
 *    DAGRT_ECUDA until dagrt_destroy;
 *  - a context is bound to one device and is NOT thread-safe (one per host
 *    thread; independent contexts on different devices run in parallel);
 *  - all device and pinned host memory is owned by the CALLER; the library
 *    never allocates or frees user data.  It owns only the streams, events
 *    and graphs it creates, released by dagrt_destroy.
 */
#ifndef DAGRT_H
#define DAGRT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dagrt_status;
enum {
  DAGRT_OK = 0,
  DAGRT_EINVAL = -1,    /* bad argument (null pointer, bad size, range out of bounds) */
  DAGRT_ENOTFOUND = -2, /* unknown or stale array / kernel handle or name */
  DAGRT_EALIAS = -3,    /* device range overlaps a registered array (no aliasing, L400-404) */
  DAGRT_ESIG = -4,      /* signature parse error or argument kind/count mismatch */
  DAGRT_ESTATE = -5,    /* call not valid in the current state (e.g. map without mirror) */
  DAGRT_ECUDA = -6,     /* CUDA runtime error (sticky) */
  DAGRT_ENOMEM = -7     /* host allocation failure */
};

typedef struct dagrt_ctx_s* dagrt_ctx;
/* Array handle: {index:32 | generation:32}; 0 is never a valid handle. */
typedef uint64_t dagrt_array;
typedef uint32_t dagrt_kernel;

/* Scheduling policy (L559-569): the original GrCUDA scheduler is serial and
 * synchronous (the baseline); the paper's scheduler is parallel and async.
 * DAGRT_PARALLEL_SINGLE_STREAM is the paper's "simpler policy" (L650-654,
 * SURVEY §8(f) f4): parallel and async with the same DAG, but every vertex
 * that has parents goes on the stream of its lowest-id parent ("schedule
 * all children on a single stream"), fewer streams and events; roots still
 * take the first empty stream in FIFO order, else a new one. */
enum { DAGRT_PARALLEL_ASYNC = 0, DAGRT_SERIAL_SYNC = 1, DAGRT_PARALLEL_SINGLE_STREAM = 2 };
/* Backend: the CUDA runtime, or a recorder that performs no device work
 * (for scheduler tests on machines without a GPU). */
enum { DAGRT_BACKEND_CUDA = 0, DAGRT_BACKEND_RECORD = 1 };
/* Host access modes for dagrt_host_map. */
enum { DAGRT_R = 1, DAGRT_W = 2, DAGRT_RW = 3 };

typedef struct {
  int32_t policy;      /* DAGRT_PARALLEL_ASYNC, DAGRT_SERIAL_SYNC or DAGRT_PARALLEL_SINGLE_STREAM */
  int32_t prefetch;    /* 1: H2D of host-newer read arguments on an in-order side copy
                          stream, overlapped with compute (L356-366, L662-664);
                          0: the copy is issued on the consumer's own stream */
  int32_t max_streams; /* 0 = unlimited; otherwise cap on compute streams */
  int32_t record_dag;  /* 1: keep vertices/edges/trace for dagrt_dag_export/dagrt_trace_export */
  int32_t backend;     /* DAGRT_BACKEND_CUDA or DAGRT_BACKEND_RECORD */
  int32_t graph_cache; /* 1: deferred submission + batch cache replayed as CUDA graphs
                          (SURVEY §8(f) f1): launches are buffered until the next host
                          synchronisation; a batch seen again is replayed with one
                          cudaGraphLaunch.  Dependencies are still inferred per launch. */
} dagrt_config;

typedef struct { uint32_t x, y, z; } dagrt_dim3;

/* One kernel argument: an array handle for pointer parameters, else a scalar
 * passed by value (scalars are "passed by copy, ignored for dependencies",
 * Fig. 4 note L450-451). */
typedef union {
  dagrt_array array;
  int32_t i32;
  int64_t i64;
  float f32;
  double f64;
} dagrt_arg;

/* ---------------------------------------------------------------- context */

/* Create a context on CUDA device `device` (ignored by the RECORD backend).
 * cfg may be NULL (defaults: parallel-async, prefetch on, unlimited streams,
 * no DAG recording, CUDA backend).  *out receives the context. */
dagrt_status dagrt_create(int device, const dagrt_config* cfg, dagrt_ctx* out);
/* Drain all work (full barrier), free the library's streams/events/graphs
 * and the context.  ctx may be NULL.  Use after destroy is undefined. */
dagrt_status dagrt_destroy(dagrt_ctx ctx);
/* Message for the last non-OK status of ctx ("" if none). */
const char* dagrt_last_error(dagrt_ctx ctx);

/* ---------------------------------------------------------------- arrays */

/* Register `bytes` of caller-owned device memory at `dev` as one array
 * (GrCUDA's managed array, L400-404, L505-507).  `host_pinned` (nullable)
 * is an optional caller-owned pinned host mirror of the same size used for
 * host accesses and transfers.  The array starts with the device copy valid
 * (the mirror is considered stale).  Overlap with a registered array ->
 * DAGRT_EALIAS.  bytes may be 0.  *out receives the handle. */
dagrt_status dagrt_array_register(dagrt_ctx ctx, void* dev, void* host_pinned, size_t bytes,
                                  dagrt_array* out);
/* Wait for the array's in-flight users, then forget it (the caller frees the
 * memory afterwards).  The handle becomes stale (DAGRT_ENOTFOUND). */
dagrt_status dagrt_array_unregister(dagrt_ctx ctx, dagrt_array a);
/* Register UNIFIED (managed) memory, cudaMallocManaged by the caller, as an
 * array: one pointer valid on host and device.  The UM mode of the paper's
 * GrCUDA (§V-C): with cfg.prefetch = 1 a host-newer array read by a
 * kernel is moved with cudaMemPrefetchAsync (on the copy stream, like an
 * H2D prefetch); with prefetch = 0 nothing is issued and the kernel's page
 * faults migrate the pages ("disabling automatic prefetching ... turns the
 * page fault controller into the main bottleneck", L904-907).  Host reads and
 * writes wait on the DAG exactly as with a mirror, then access the memory
 * directly (no copy).  Registering a managed array turns the graph cache of
 * the context off (prefetches are not graph nodes). */
dagrt_status dagrt_array_register_managed(dagrt_ctx ctx, void* ptr, size_t bytes, dagrt_array* out);
/* Conveniences for callers without a CUDA binding of their own (the only
 * memory functions of the library; not used on the product path):
 * cudaMallocManaged / cudaFree, and moving the pages of [p, p+bytes) to the
 * host (cudaMemPrefetchAsync to the CPU + synchronize) so that the next GPU
 * access must migrate them again. */
dagrt_status dagrt_managed_alloc(size_t bytes, void** p);
dagrt_status dagrt_managed_free(void* p);
dagrt_status dagrt_managed_to_host(void* p, size_t bytes);
/* Device pointer of a registered array (for the caller's own bookkeeping). */
dagrt_status dagrt_array_device_ptr(dagrt_ctx ctx, dagrt_array a, void** dev);

/* ---------------------------------------------------------------- kernels */

/* Declare a kernel: `global_fn` is a __global__ function symbol compiled for
 * sm_100a (may be NULL with the RECORD backend), `name` a label, `signature`
 * one comma-separated token per parameter (L431-433, L668-677):
 *   "const ptr" | "in ptr"   read-only pointer   (prefetched)
 *   "ptr" | "inout ptr"      modified pointer    (prefetched)   -- unannotated = modified
 *   "out ptr"                modified pointer, overwritten entirely (not prefetched)
 *   "sint32" | "sint64" | "float" | "double"   scalar by value, no dependency
 * At most 16 parameters.  Parse error -> DAGRT_ESIG. */
dagrt_status dagrt_kernel_register(dagrt_ctx ctx, const void* global_fn, const char* name,
                                   const char* signature, dagrt_kernel* out);
/* Find a kernel by name: user-registered ones, then the built-in sm_100a
 * benchmark kernels of the library (list: dagrt_builtin_count/_name). */
dagrt_status dagrt_kernel_lookup(dagrt_ctx ctx, const char* name, dagrt_kernel* out);
/* Parameter kinds of kernel k: kinds[i] = 0 sint32, 1 sint64, 2 const ptr,
 * 3 mutable ptr (prefetched), 4 out ptr, 5 float, 6 double.
 * *n: capacity in, count out. */
dagrt_status dagrt_kernel_signature(dagrt_ctx ctx, dagrt_kernel k, int32_t* kinds, int32_t* n);
/* Name of kernel handle k (built-in, registered or library-call pseudo-kernel);
 * NULL if k is not a handle of ctx.  Owned by the context. */
const char* dagrt_kernel_name(dagrt_ctx ctx, dagrt_kernel k);
int32_t dagrt_builtin_count(void);
const char* dagrt_builtin_name(int32_t i);
const char* dagrt_builtin_signature(int32_t i);

/* History-driven launch configuration (the scheduler keeps
 * "historical information" about computations, L502-504, and the paper names
 * the automatic choice of launch parameters as future work, L1502-1504 /
 * Fig. 7).  Registers n candidate configurations for kernel k;
 * afterwards a dagrt_launch of k with grid = {0, 0, 0} ("auto") takes one of
 * them: while exploring, the candidates are used in turn, `trials` times
 * each, every such launch bracketed by timing events on its own stream; the
 * timings are collected without blocking at later host synchronisations, and
 * once every candidate has `trials` samples the one with the lowest median
 * time is used from then on.  History is kept per (kernel, key), key = a hash
 * of the launch's scalar arguments (the problem size), so each size is tuned
 * on its own.  The DAG does not depend on it (launch configurations take no
 * part in dependency inference).  With the graph cache on, exploration is
 * suspended (auto launches use the best configuration known so far, else the
 * first candidate).  Candidates are copied; n <= 16, trials >= 1. */
typedef struct {
  dagrt_dim3 grid, block;
  uint32_t smem;
} dagrt_launch_config;
dagrt_status dagrt_kernel_autotune(dagrt_ctx ctx, dagrt_kernel k, const dagrt_launch_config* candidates, int32_t n,
                                   int32_t trials);
/* History of kernel k for the scalar-argument key of its LAST auto launch:
 * *chosen = index of the selected candidate (-1 while exploring), ms[i] = the
 * median time of candidate i so far (-1 if unsampled), *n: capacity in, count
 * out. */
dagrt_status dagrt_autotune_state(dagrt_ctx ctx, dagrt_kernel k, int32_t* chosen, double* ms, int32_t* n);

/* ---------------------------------------------------------------- launch */

/* Launch kernel k with `nargs` arguments (count and kinds must match the
 * signature, else DAGRT_ESIG).  Never blocks the host under the parallel
 * policy (L564-569): builds the computational element (L388-396), computes
 * its parents from the dependency sets of active computations (L408-431,
 * L490-491), picks a stream (L570-582, L647-650), makes the stream wait on
 * the events of parents running on other streams (L546-553), prefetches
 * host-newer read arguments on the copy stream (L356-366), launches, and
 * records the vertex's event.  Under DAGRT_SERIAL_SYNC the launch and any
 * copy run on one stream, each followed by a stream synchronize (L560-569). */
dagrt_status dagrt_launch(dagrt_ctx ctx, dagrt_kernel k, dagrt_dim3 grid, dagrt_dim3 block,
                          uint32_t smem, const dagrt_arg* args, int32_t nargs);

/* The same call with its arguments in one caller-owned descriptor (read
 * during the call only): identical semantics to dagrt_launch, for bindings
 * whose per-argument marshalling cost is comparable to the launch itself
 * (one pointer instead of seven arguments per call from Python). */
typedef struct {
  dagrt_kernel kernel;
  dagrt_dim3 grid, block;
  uint32_t smem;
  int32_t nargs;
  const dagrt_arg* args;
} dagrt_launch_desc;
dagrt_status dagrt_launch_prepared(dagrt_ctx ctx, const dagrt_launch_desc* d);
/* n consecutive launches descs[0..n-1] in program order: exactly the same as
 * n dagrt_launch_prepared calls (each is its own DAG vertex, dependencies are
 * inferred launch by launch); stops at the first failing launch and returns
 * its status (the launches before it have been issued).  For bindings whose
 * per-call cost is comparable to a launch (Python: ~2.5 us per call on the
 * B200 box host). */
dagrt_status dagrt_launch_batch(dagrt_ctx ctx, const dagrt_launch_desc* descs, int32_t n);

/* A LIBRARY CALL as a DAG vertex (L516-519: besides kernels, "library
 * functions" executed on the GPU are computational elements whose argument
 * modes the scheduler uses).  The vertex is scheduled exactly like a kernel
 * (dependencies from `arrays` with modes[i] in DAGRT_R / DAGRT_W (overwritten
 * whole: not prefetched) / DAGRT_RW, stream choice, event wiring, prefetch);
 * instead of a kernel launch the scheduler calls fn(stream, user) on the host
 * with the CUDA stream (cudaStream_t) it picked.  fn must enqueue all its GPU
 * work for these arrays on that stream, must not synchronise, and returns 0
 * (nonzero: DAGRT_EINVAL, the vertex is not recorded).  `name` labels the
 * vertex in dagrt_dag_export (a pseudo-kernel per distinct name).  Ownership:
 * fn and user stay the caller's; fn is called during this call only.  With
 * the graph cache on, pending deferred work is flushed first (a host callback
 * cannot be captured). */
typedef int32_t (*dagrt_library_fn)(void* stream, void* user);
dagrt_status dagrt_launch_library(dagrt_ctx ctx, dagrt_library_fn fn, void* user, const char* name,
                                  const dagrt_array* arrays, const int32_t* modes, int32_t n);

/* ---------------------------------------------------------------- host access */

/* Host read of bytes [off, off+bytes) of array a into dst (L505-516): if the
 * access conflicts with active GPU work it becomes a DAG vertex and the host
 * waits on exactly the conflicting computations' events, retiring them and
 * their ancestors (L526-528, L553-556); then the range is copied D2H if the
 * device copy is newer (via the mirror when one is registered).  A
 * non-conflicting access runs immediately and is not recorded (L512-516). */
dagrt_status dagrt_host_read(dagrt_ctx ctx, dagrt_array a, size_t off, size_t bytes, void* dst);
/* Host write of [off, off+bytes) from src: waits on the active readers since
 * the last writer, else on the last writer (reading D6), then writes the
 * mirror (marking the host copy newer; the next GPU reader pulls it) or,
 * without a mirror, copies H2D synchronously.  A partial write of a
 * device-newer mirrored array first pulls the whole array D2H. */
dagrt_status dagrt_host_write(dagrt_ctx ctx, dagrt_array a, size_t off, size_t bytes,
                              const void* src);
/* Whole-array host access through the pinned mirror (DAGRT_ESTATE without
 * one): access R syncs like host_read and makes the mirror current; W syncs
 * like host_write and marks the host copy newer (the caller writes through
 * *host_ptr until dagrt_host_unmap).  RW does both. */
dagrt_status dagrt_host_map(dagrt_ctx ctx, dagrt_array a, int32_t access, void** host_ptr);
dagrt_status dagrt_host_unmap(dagrt_ctx ctx, dagrt_array a);
/* Full barrier (build-only API, reading D6b): waits for all streams and
 * retires every active computation.  Records no vertex. */
dagrt_status dagrt_sync(dagrt_ctx ctx);

/* ---------------------------------------------------------------- introspection */

typedef struct {
  uint32_t id;     /* vertex id = order of recording */
  uint32_t kind;   /* 0 kernel, 1 host access */
  uint32_t kernel; /* kernel handle (kind 0) */
  int32_t stream;  /* compute stream index (0-based, creation order); -1 for host */
  dagrt_array array; /* accessed array (kind 1), else 0 */
} dagrt_vertex_info;

typedef struct {
  uint32_t parent, child;
  dagrt_array array; /* the argument causing the dependency (one row per label, L218-220) */
} dagrt_edge_info;

/* Copy out the DAG recorded since the last dagrt_dag_clear (needs
 * record_dag=1).  *nv / *ne: capacity in, count out; NULL arrays query the
 * counts; insufficient capacity -> DAGRT_EINVAL with the counts set.  The
 * scheduler itself only ever keeps the active frontier (L495-501). */
dagrt_status dagrt_dag_export(dagrt_ctx ctx, dagrt_vertex_info* v, uint32_t* nv,
                              dagrt_edge_info* e, uint32_t* ne);
dagrt_status dagrt_dag_clear(dagrt_ctx ctx);

/* Backend operation trace (record_dag=1), for event-wiring and transfer checks. */
enum {
  DAGRT_OP_LAUNCH = 1,      /* a = vertex, b = kernel, stream */
  DAGRT_OP_RECORD = 2,      /* a = vertex, stream: event of vertex a recorded */
  DAGRT_OP_WAIT = 3,        /* stream waits on the event of vertex a */
  DAGRT_OP_H2D = 4,         /* a = array index, bytes, stream (-2 = copy stream) */
  DAGRT_OP_D2H = 5,         /* a = array index, bytes */
  DAGRT_OP_EVENT_SYNC = 6,  /* host waits on the event of vertex a */
  DAGRT_OP_STREAM_SYNC = 7, /* host waits on stream */
  DAGRT_OP_WAIT_COPY = 8    /* stream waits on the H2D copy event of array a */
};
typedef struct {
  int32_t op;
  int32_t stream; /* compute stream index, -2 copy stream, -1 none */
  int64_t a, b;
  uint64_t bytes;
} dagrt_trace_op;
dagrt_status dagrt_trace_export(dagrt_ctx ctx, dagrt_trace_op* ops, uint32_t* n);

typedef struct {
  uint64_t launches;           /* kernel launches */
  uint64_t vertices;           /* recorded vertices (kernels + conflicting host accesses) */
  uint64_t host_vertices;
  uint64_t edges;              /* (parent, child) pairs */
  uint64_t cross_stream_waits; /* cudaStreamWaitEvent on vertex events */
  uint64_t copy_waits;         /* cudaStreamWaitEvent on copy events */
  uint64_t streams;            /* compute streams created */
  uint64_t events_created;
  uint64_t h2d_bytes, d2h_bytes, h2d_copies, d2h_copies;
  uint64_t host_syncs;         /* host-blocking waits (event or stream) */
  uint64_t sched_ns;           /* host ns spent inside dagrt_launch */
  uint64_t graph_replays;      /* batches replayed from the graph cache */
  uint64_t graph_captures;     /* batches captured into a new graph */
  uint64_t eager_batches;      /* batches issued eagerly (first sighting) */
  /* breakdown of sched_ns (host ns inside dagrt_launch): time in the CUDA
   * enqueue calls themselves; the rest is the scheduler's own bookkeeping */
  uint64_t launch_ns;          /* cuLaunchKernel / cudaLaunchCooperativeKernel */
  uint64_t record_ns;          /* cudaEventRecord of the vertex event */
  uint64_t wait_ns;            /* cudaStreamWaitEvent (cross-stream and copy waits) + H2D enqueue */
  /* bounded state: the vertex table holds the current epoch only (it is
   * dropped whenever the active frontier empties) */
  uint64_t table_vertices;     /* vertex records held now */
  uint64_t epoch_base;         /* global id of the first record held */
  uint64_t max_readers;        /* longest reader list of any live array now */
  uint64_t um_prefetch_bytes;  /* managed arrays: bytes moved by cudaMemPrefetchAsync */
  uint64_t um_fault_bytes;     /* managed arrays: host-newer bytes left to GPU page faults */
} dagrt_stats_t;
/* Copy min(size, sizeof(dagrt_stats_t)) bytes of the counters to out. */
dagrt_status dagrt_stats(dagrt_ctx ctx, void* out, size_t size);
dagrt_status dagrt_stats_reset(dagrt_ctx ctx);
/* Number of compute streams the context has created. */
dagrt_status dagrt_stream_count(dagrt_ctx ctx, int32_t* n);
/* The cudaStream_t of compute stream i (as void*), e.g. for profiling marks. */
dagrt_status dagrt_stream_handle(dagrt_ctx ctx, int32_t i, void** stream);

/* Kernel timing on the launching stream: while enabled for kernel k, every
 * launch of k is bracketed by two timing events recorded on the stream the
 * scheduler put it on (2 extra cudaEventRecord per launch). */
dagrt_status dagrt_profile_enable(dagrt_ctx ctx, dagrt_kernel k, int32_t on);
/* Wait for the recorded launches of k and report: *count launches, *sum_ms
 * the sum of their durations, *busy_ms the length of the union of their
 * [start, end] intervals (time during which at least one launch of k was
 * running; concurrent launches overlap).  Clears the records. */
dagrt_status dagrt_profile_collect(dagrt_ctx ctx, dagrt_kernel k, int32_t* count, double* sum_ms,
                                   double* busy_ms);

/* Execution timeline (schedule evidence, the paper's Fig. 10 / L1265-1291):
 * while enabled, every kernel launch and every H2D/D2H copy issued by the
 * scheduler is bracketed by timing events on its own stream.  Export waits
 * for them and returns one record per item, times in ms relative to the
 * first recorded item, then clears the records. */
typedef struct {
  int32_t kind;    /* 0 kernel, 1 H2D copy, 2 D2H copy */
  int32_t stream;  /* compute stream index, -2 copy stream, -3 serial stream, -5 D2H stream */
  int64_t vertex;  /* vertex id (kernels; H2D: consuming vertex; D2H: -1) */
  int64_t id;      /* kernel handle (kind 0) or array index (copies) */
  uint64_t bytes;  /* copy size (copies) */
  double start_ms, end_ms;
} dagrt_timeline_rec;
dagrt_status dagrt_timeline_enable(dagrt_ctx ctx, int32_t on);
dagrt_status dagrt_timeline_export(dagrt_ctx ctx, dagrt_timeline_rec* recs, uint32_t* n);

/* ---------------------------------------------------------------- baselines */

/* Direct launch on a caller-given cudaStream_t with no scheduling at all
 * (arrays resolved to device pointers only).  For the hand-written schedules
 * the paper compares against (CUDA Graphs, L1057-1070). */
dagrt_status dagrt_launch_raw(dagrt_ctx ctx, dagrt_kernel k, dagrt_dim3 grid, dagrt_dim3 block,
                              uint32_t smem, const dagrt_arg* args, int32_t nargs, void* stream);

/* Hand-built CUDA graph with MANUAL dependencies ("Graph API + manual
 * dependencies", L1062-1067): nodes are added with the explicit list of
 * earlier node ids they depend on; nothing is inferred. */
typedef struct dagrt_graph_s* dagrt_graph;
dagrt_status dagrt_graph_create(dagrt_ctx ctx, dagrt_graph* g);
/* Kernel node; deps are node ids returned by earlier add calls. */
dagrt_status dagrt_graph_add_kernel(dagrt_ctx ctx, dagrt_graph g, dagrt_kernel k, dagrt_dim3 grid,
                                    dagrt_dim3 block, uint32_t smem, const dagrt_arg* args,
                                    int32_t nargs, const uint32_t* deps, int32_t ndeps,
                                    uint32_t* node);
/* Copy node between an array's device memory and its pinned mirror:
 * dir 0 = H2D, 1 = D2H, bytes [off, off+bytes). */
dagrt_status dagrt_graph_add_copy(dagrt_ctx ctx, dagrt_graph g, dagrt_array a, int32_t dir,
                                  size_t off, size_t bytes, const uint32_t* deps, int32_t ndeps,
                                  uint32_t* node);
/* D2H copy node from array a's device bytes [off, off+bytes) into
 * caller-owned PINNED host memory dst (which must stay valid while the graph
 * exists): the graph's equivalent of a host read of a sink (resident mode
 * reads one element per sink), so that every compared schedule
 * ends with the host holding the outputs. */
dagrt_status dagrt_graph_add_read(dagrt_ctx ctx, dagrt_graph g, dagrt_array a, size_t off,
                                  size_t bytes, void* dst, const uint32_t* deps, int32_t ndeps,
                                  uint32_t* node);
dagrt_status dagrt_graph_instantiate(dagrt_ctx ctx, dagrt_graph g);
/* Launch the instantiated graph on the context's graph stream and wait for it. */
dagrt_status dagrt_graph_run(dagrt_ctx ctx, dagrt_graph g, int32_t wait);
dagrt_status dagrt_graph_destroy(dagrt_ctx ctx, dagrt_graph g);

/* ---------------------------------------------------------------- multi-GPU placement (f2)
 *
 * The paper's future work (L1499-1502: "compute data location and migration
 * costs at run time" to use several GPUs).  A multi-context drives one
 * dagrt_ctx per SLOT (a CUDA device; the same device may back several slots,
 * which is how a one-GPU box exercises the cross-slot path) from ONE host
 * thread.  Every launch is a vertex of the DAG of the slot it is PLACED on;
 * the per-slot schedulers infer dependencies, streams and events as for a
 * single GPU.  Arrays are multi-arrays: a home copy (caller-owned), replicas
 * on other slots (allocated by the library on first use, freed by
 * dagrt_multi_destroy) and an optional pinned host mirror, with a validity
 * set over {slots, host}.  A launch on slot d whose read arguments are not
 * valid on d first migrates them, as library-call vertices (dagrt_launch_library):
 *   slot -> slot: "migrate_pre" on d (mode W: waits d's users of the old
 *     replica, records an event), "migrate_out" on the source slot (mode R:
 *     after the last writer there, waits that event, cudaMemcpyPeerAsync over
 *     NVLink / NVSwitch, records a second event) and "migrate_in" on d (mode W:
 *     waits it) -- so later writers on the source wait for the copy, and
 *     readers on d for its completion: a cross-device edge is a peer copy
 *     plus cross-device events, no collective;
 *   host -> slot: "upload" on d (mode W: cudaMemcpyAsync from the mirror).
 * A kernel's writes leave only the replica it wrote valid.
 *
 * Placement: DAGRT_PLACE_DATA (default) estimates for every slot the time
 * the vertex would finish -- the slot's estimated busy time, plus the bytes
 * of read arguments not valid there over the link bandwidth they would
 * cross (host 50 GB/s, peer 700 GB/s, same device 3000 GB/s), plus the
 * vertex's own argument bytes over HBM bandwidth (6500 GB/s) -- and takes the
 * earliest (ties: the lower slot); the busy estimates reset at
 * dagrt_multi_sync.  DAGRT_PLACE_ROUND_ROBIN cycles over the slots.  A launch
 * may also force a slot (slot >= 0).  Not thread-safe, like dagrt_ctx. */
typedef struct dagrt_multi_s* dagrt_multi;
/* Multi-array handle {index:32 | generation:32}; 0 is never valid. */
typedef uint64_t dagrt_marray;
enum { DAGRT_PLACE_DATA = 0, DAGRT_PLACE_ROUND_ROBIN = 1 };
typedef struct {
  uint64_t launches;          /* kernels launched through dagrt_multi_launch */
  uint64_t migrations_peer;   /* slot -> slot array copies */
  uint64_t bytes_peer;
  uint64_t migrations_host;   /* host mirror -> slot copies */
  uint64_t bytes_host;
  uint64_t replicas;          /* replicas allocated by the library */
  uint64_t bytes_replicas;
  uint64_t per_slot[16];      /* launches placed on each slot */
} dagrt_multi_stats_t;
/* Create a multi-context over n (1..16) slots; devices[i] is slot i's CUDA
 * device (ignored by the RECORD backend); cfg as for dagrt_create (applied
 * to every slot); placement = DAGRT_PLACE_*.  Peer access is enabled between
 * the distinct devices where the hardware allows it. */
dagrt_status dagrt_multi_create(const int32_t* devices, int32_t n, const dagrt_config* cfg, int32_t placement,
                                dagrt_multi* out);
/* Waits for all work, frees the replicas, destroys the slot contexts. */
dagrt_status dagrt_multi_destroy(dagrt_multi m);
const char* dagrt_multi_last_error(dagrt_multi m);
/* The slot's own context (for introspection: dagrt_dag_export, stats). */
dagrt_status dagrt_multi_slot_ctx(dagrt_multi m, int32_t slot, dagrt_ctx* out);
/* Register caller-owned memory as a multi-array: `dev` on slot `home` (NULL:
 * the library allocates the home copy too), optional pinned host mirror.
 * The array starts valid on its home slot if `dev` was given, else on the
 * host if a mirror was given (else it is undefined until written). */
dagrt_status dagrt_multi_array_register(dagrt_multi m, int32_t home, void* dev, void* host_pinned, size_t bytes,
                                        dagrt_marray* out);
/* Device pointer of the array's copy on a slot (NULL if none yet). */
dagrt_status dagrt_multi_array_ptr(dagrt_multi m, dagrt_marray a, int32_t slot, void** dev);
/* Launch built-in or registered kernel `name` (looked up in every slot's
 * context): pointer arguments are dagrt_marray handles.  slot < 0: placed by
 * the policy; *placed (nullable) receives the slot. */
dagrt_status dagrt_multi_launch(dagrt_multi m, const char* name, dagrt_dim3 grid, dagrt_dim3 block, uint32_t smem,
                                const dagrt_arg* args, int32_t nargs, int32_t slot, int32_t* placed);
/* Host read of [off, off+bytes): from the mirror if the host copy is valid,
 * else through the context of a slot holding a valid copy (dagrt_host_read:
 * waits exactly for that copy's writer). */
dagrt_status dagrt_multi_host_read(dagrt_multi m, dagrt_marray a, size_t off, size_t bytes, void* dst);
/* Host write of [off, off+bytes) from src.  With a mirror: waits for uploads
 * still reading it, makes it current first if the write is partial, copies
 * src into it (src may be the mirror itself: the caller wrote it in place)
 * and leaves only the host copy valid.  Without a mirror: written into the
 * home copy through the home slot's context (dagrt_host_write). */
dagrt_status dagrt_multi_host_write(dagrt_multi m, dagrt_marray a, size_t off, size_t bytes, const void* src);
/* Barrier over every slot (dagrt_sync each); resets the busy estimates. */
dagrt_status dagrt_multi_sync(dagrt_multi m);
dagrt_status dagrt_multi_stats(dagrt_multi m, dagrt_multi_stats_t* out);

#ifdef __cplusplus
}
#endif
#endif /* DAGRT_H */
