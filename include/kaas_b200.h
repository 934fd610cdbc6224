/*
 * kaas_b200.h -- C ABI of the B200-native KaaS executor (libkaas_b200.so).
 *
 * The reference (arXiv 2212.08146 artifact, pkg/src/kaas) is pure Python and
 * has no native FFI; its "device" is host bytearrays driven by numpy.  Each
 * entry point below replaces one device-touching step of that path; the
 * reference call it stands in for is cited beside it.  A ctypes binding for
 * the reference's own backend/executor classes is shown in INTEGRATION.md.
 *
 * Conventions
 *   - every function returns int: 0 = ok, >0 = cudaError_t, <0 = KAAS_E_*;
 *     kaas_last_error() returns the thread-local message of the last failure.
 *   - device pointers, streams and events travel as uint64_t handles.
 *   - no torch types; plain pointers and sizes only.
 *   - thread safety: calls for different devices / streams may run
 *     concurrently (one host worker thread per device is the intended use).
 *   - ownership: the caller owns every allocation and frees it; the library
 *     keeps only per-stream scratch (reductions, cGEMM operand staging),
 *     released by kaas_stream_destroy.
 */
#ifndef KAAS_B200_H
#define KAAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define KAAS_OK 0
#define KAAS_E_INVALID (-1)     /* bad argument (null pointer, bad id)       */
#define KAAS_E_ARITY (-2)       /* literal tags / buffer count mismatch      */
#define KAAS_E_BOUNDS (-3)      /* launch would touch bytes past a buffer    */
#define KAAS_E_UNKNOWN_KERNEL (-4)
#define KAAS_E_UNSUPPORTED (-5) /* e.g. device is not sm_100               */

/* ---- kernel ids (reference ids in pkg/src/kaas/backend.py:236-243) ----- */
#define KAAS_K_VECTOR_ADD 1  /* backend.py:153-160  (i32 n; X, Y, OUT)          */
#define KAAS_K_SAXPY 2       /* backend.py:163-171  (i32 n, f32 a; X, Y, OUT)   */
#define KAAS_K_MATMUL 3      /* backend.py:174-189  (i32 n,m,k; A, B, OUT)      */
#define KAAS_K_REDUCE_SUM 4  /* backend.py:192-202  (i32 n; X, OUT)             */
#define KAAS_K_FILL 5        /* backend.py:205-211  (i32 n, f32 v; OUT)         */
#define KAAS_K_CGEMM 6       /* new: (i32 n,m,k; A, B, C) complex64, 4M x 3xFP16 */
#define KAAS_K_JACOBI 7      /* new: (i32 n; A, b, x_in, x_out, resid)         */

/* kaas_launch_desc.flags for KAAS_K_CGEMM: prepared-operand cache.  ptrs[3] /
 * ptrs[4] (sizes[3] / sizes[4]) then hold the executor-owned buffers for the
 * scaled 3xFP16-split A ([A_hi; A_lo] 2*n*ldk fp16, then n u32 row
 * max-bits: 4*n*ldk + 4*n bytes) and 4M-expanded, transposed, split B
 * ([Bt_hi; Bt_lo] 4*m*ldk fp16, then m u32 column max-bits: 8*m*ldk + 4*m
 * bytes), ldk = 2k rounded up to 64.  USE:
 * the buffer already holds them; FILL: compute them into it (else the
 * per-stream scratch is used and nothing is kept). */
#define KAAS_F_CG_A_USE 1
#define KAAS_F_CG_B_USE 2
#define KAAS_F_CG_A_FILL 4
#define KAAS_F_CG_B_FILL 8
/* kaas_launch_desc.flags for KAAS_K_MATMUL: ptrs[3] / sizes[3] hold an
 * executor-owned buffer for B transposed ([m][k] f32, 4*m*k bytes) -- the
 * prepared form of a const weight.  USE: it holds Bt; FILL: build it first. */
#define KAAS_F_MM_BT_USE 16
#define KAAS_F_MM_BT_FILL 32

/* literal tags, protocol.py:27 LITERAL_TYPES order */
#define KAAS_LIT_I32 0
#define KAAS_LIT_I64 1
#define KAAS_LIT_F32 2
#define KAAS_LIT_F64 3

typedef struct kaas_literal {
  int32_t tag;
  int32_t reserved;
  int64_t i; /* integer payload (i32/i64)            */
  double f;  /* float payload (f32 rounded on device) */
} kaas_literal;

#define KAAS_MAX_LITS 4
#define KAAS_MAX_ARGS 8

/* One kernel invocation (protocol.py:129-134 KernelInvocation, with the
 * buffer names already resolved to device pointers by the executor). */
typedef struct kaas_launch_desc {
  int32_t kernel;
  int32_t n_lits;
  int32_t n_args;
  int32_t flags;
  uint32_t dims[6]; /* grid_x, grid_y, grid_z, block_x, block_y, block_z */
  uint32_t reserved[2];
  kaas_literal lits[KAAS_MAX_LITS];
  uint64_t ptrs[KAAS_MAX_ARGS];
  uint64_t sizes[KAAS_MAX_ARGS];
} kaas_launch_desc;

typedef struct kaas_device_info {
  int32_t ordinal;
  int32_t sm_count;
  int32_t cc_major;
  int32_t cc_minor;
  uint64_t total_mem;
  uint64_t l2_bytes;
  int32_t max_smem_per_block;
  int32_t clock_khz;
  char name[128];
} kaas_device_info;

/* ---- errors / discovery ------------------------------------------------- */
int kaas_last_error(char *buf, size_t len);
int kaas_version(int *major, int *minor);
int kaas_device_count(int *n);
/* Set up device `dev` (memory pool that keeps freed pages, peer maps). */
int kaas_init_device(int dev);
int kaas_device_info_get(int dev, kaas_device_info *out);
/* Total kernels this library has launched (all devices) -- bench evidence. */
int kaas_launch_counter(uint64_t *out);
/* Device health after a failed call: 0, or the sticky CUDA error (the
 * executor is then poisoned and the router stops placing requests on it;
 * replaces the worker's exception path, service.py:71-78). */
int kaas_device_check(int dev);
/* Fault injection for tests (genreq.py:190-243 injects request faults; this
 * injects a device fault): enqueues a kernel that traps on `stream`. */
int kaas_inject_fault(uint64_t stream);

/* ---- streams / events (executor request lifecycle, executor.py:320-387) */
int kaas_stream_create(int dev, int priority, uint64_t *stream);
int kaas_stream_destroy(uint64_t stream);
int kaas_stream_sync(uint64_t stream);
int kaas_event_create(int dev, int timing, uint64_t *event);
int kaas_event_destroy(uint64_t event);
int kaas_event_record(uint64_t event, uint64_t stream);
int kaas_stream_wait_event(uint64_t stream, uint64_t event);
int kaas_event_sync(uint64_t event);
int kaas_event_query(uint64_t event, int *done);
int kaas_event_elapsed_ms(uint64_t start, uint64_t end, float *ms);
/* n (start, end) pairs in one crossing (a request's device-timing spans) */
int kaas_event_elapsed_many(int n, const uint64_t *starts, const uint64_t *ends, float *ms);

/* ---- device memory: DeviceBuffer.__init__ (executor.py:63-72) ---------- */
int kaas_malloc_async(uint64_t stream, uint64_t bytes, uint64_t *dptr);
int kaas_free_async(uint64_t stream, uint64_t dptr);
/* zero-fill of outputs / ephemerals (executor.py:70 bytearray zeros) */
int kaas_memset_async(uint64_t dptr, int value, uint64_t bytes, uint64_t stream);

/* ---- pinned host memory (MemoryStore payloads, store.py:65-98) --------- */
int kaas_host_alloc(uint64_t bytes, void **ptr);
int kaas_host_free(void *ptr);
int kaas_host_register(void *ptr, uint64_t bytes);
int kaas_host_unregister(void *ptr);

/* ---- copies: DeviceBuffer.load / snapshot (executor.py:78-82) ---------- */
int kaas_memcpy_h2d_async(uint64_t dst, const void *src, uint64_t bytes, uint64_t stream);
int kaas_memcpy_d2h_async(void *dst, uint64_t src, uint64_t bytes, uint64_t stream);
int kaas_memcpy_d2d_async(uint64_t dst, uint64_t src, uint64_t bytes, uint64_t stream);
/* NVLink peer fill of a cache entry another GPU already holds (new).
 * kaas_enable_peer(dev, peer): `dev` may read `peer`'s memory, including
 * allocations from `peer`'s stream-ordered pool (cudaMemPoolSetAccess). */
int kaas_enable_peer(int dev, int peer);
int kaas_can_access_peer(int dev, int peer, int *can);
int kaas_memcpy_p2p_async(uint64_t dst, int dst_dev, uint64_t src, int src_dev,
                          uint64_t bytes, uint64_t stream);

/* ---- kernels: SimulatedBackend.launch (backend.py:258-266) ------------- */
/* Bounds are re-checked here (backend.py:137-150 _extent/_f32_view rules);
 * a violation returns KAAS_E_BOUNDS and enqueues nothing. */
int kaas_launch(int dev, uint64_t stream, const kaas_launch_desc *desc);
/* The invocation loop of Executor.execute (executor.py:356-369) in one
 * crossing: descs run in order on `stream`.  All descriptors are validated
 * before the first enqueue.  Runs of KAAS_K_JACOBI sweeps that ping-pong
 * their x buffers are fused into one persistent multi-sweep launch. */
int kaas_launch_batch(int dev, uint64_t stream, const kaas_launch_desc *descs, int n);

/* Progressive write-back (new; overlaps Executor.execute's flush loop,
 * executor.py:371-380, with the kernel that produces the flushed buffer).
 * Copies bytes [0, bytes) of descs[desc_index].ptrs[arg_index] into the
 * pinned host_dst on out_stream, ordered after that kernel.  cGEMM outputs
 * are streamed per finished row panel while later tiles still compute
 * (device-side panel counters + cuStreamWaitValue32); other kernels copy
 * once the kernel completes.  The descriptor must be the last in the batch
 * that writes that buffer. */
typedef struct kaas_stream_out {
  int32_t desc_index;
  int32_t arg_index;
  uint64_t out_stream;
  void *host_dst;
  uint64_t bytes;
} kaas_stream_out;
int kaas_launch_batch_ex(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                         const kaas_stream_out *outs, int n_outs);
/* kaas_launch_batch with a caller-chosen memo key: a nonzero key promises
 * that `descs` has exactly the content of the last call on this stream that
 * used the same key, so a fused Jacobi chain is relaunched from its cached
 * parameters without re-parsing the descriptors (key 0 = no memo). */
int kaas_launch_batch_memo(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                           uint64_t memo_key);
/* kaas_launch_batch_memo with the request's stream plumbing in the same
 * crossing (the executor's launch step, executor.py:356-369): when
 * join_event != 0 it is recorded on join_stream (the fills' copy stream) and
 * `stream` waits for it; ev_start / ev_end (0 = none) are recorded on
 * `stream` right before / after the launches (the request's kernel span).
 * `outs` (as kaas_launch_batch_ex): the final contents of those buffers are
 * in host_dst once ev_end has completed -- a fused Jacobi chain writes its
 * last sweep's x_out / resid there from the kernel, anything else is copied
 * on the spec's out_stream after the batch (pass `stream` itself as the
 * out_stream so that ev_end covers those copies). */
int kaas_launch_batch_timed(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                            uint64_t memo_key, uint64_t join_stream, uint64_t join_event,
                            uint64_t ev_start, uint64_t ev_end, const kaas_stream_out *outs,
                            int n_outs);

#ifdef __cplusplus
}
#endif
#endif /* KAAS_B200_H */
