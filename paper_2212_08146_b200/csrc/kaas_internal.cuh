// Internal declarations shared by the C-ABI layer and the kernel files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/kaas_b200.h"

namespace kaas {

// ---- developer switches ------------------------------------------------------
// A/B switches read from the environment exist only in developer builds
// (make dev -> libkaas_b200_dev.so, -DKAAS_DEV).  The product library never
// reads the environment: every switch folds to its default at compile time.
#ifdef KAAS_DEV
#include <cstdlib>
#define KAAS_DEV_ENV(name) std::getenv(name)
#else
#define KAAS_DEV_ENV(name) (static_cast<const char *>(nullptr))
#endif

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define KAAS_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return ::kaas::cuda_fail(_e, #call); \
  } while (0)

// ---- per-stream scratch (outside the cache ledger) ------------------------
// Each executor stream owns its own scratch so two executors sharing a GPU
// never race on reduction partials or cGEMM operand staging.
struct StreamScratch {
  int dev = 0;
  // Jacobi: per-block residual partials + arrival ticket + grid barrier words
  float *jac_partials = nullptr;    // [kMaxJacobiBlocks]
  unsigned *jac_sync = nullptr;     // [4]: ticket, barrier count, barrier gen, pad
  // cGEMM operand staging (A_lo, B_exp^T hi, B_exp^T lo), grown on demand
  void *cg_buf = nullptr;
  size_t cg_bytes = 0;
  // per-row-panel tile completion counters for progressive write-back
  unsigned *panel_done = nullptr;  // [kMaxPanels], plain cudaMalloc (stream mem-op target)
  // Jacobi column kernel: x published as (value, tag) words, ping-pong
  unsigned long long *jac_xt = nullptr;  // [2][kJacTaggedMaxN], zeroed at creation
  unsigned jac_tag = 1;                  // next launch's tag base (host side, stream-ordered)
  unsigned jac_sync_base = 0;            // value of the monotonic barrier counter jac_sync[3]
  // bit-exact matmul: B transposed for one launch when no prepared copy exists
  void *mm_buf = nullptr;
  size_t mm_bytes = 0;
  // memoised fused Jacobi chain (kaas_launch_batch_memo): the built launch
  // parameters of the last single-launch chain, keyed by the caller's key
  uint64_t jac_memo_key = 0;
  void *jac_memo = nullptr;  // owned; freed by free_jacobi_memo
  // cGEMM write-back ordering events, created on first use, reused per launch
  cudaEvent_t cg_ev_ready = nullptr, cg_ev_done = nullptr;
  // invocation-run kernel (runs.cu): per-task arrival counters, monotonic
  // across launches, and the host's running expectation of each
  unsigned *run_done = nullptr;  // [kRunMaxTasks]
  std::vector<uint32_t> run_expect;
};
constexpr int kJacTaggedMaxN = 4096;
constexpr int kMaxPanels = 1024;

// Progressive write-back of one kernel output (see kaas_launch_batch_ex).
struct ProgressiveOut {
  cudaStream_t out_stream;
  void *host;
  uint64_t bytes;  // bytes of the output buffer to copy
};
constexpr int kMaxJacobiBlocks = 4096;

StreamScratch *scratch_for(cudaStream_t s);
int ensure_cgemm_scratch(StreamScratch *sc, cudaStream_t s, size_t bytes);
int ensure_matmul_scratch(StreamScratch *sc, cudaStream_t s, size_t bytes);

struct DeviceProps {
  int sm_count = 148;
  int max_smem_optin = 227 * 1024;
  int cc_major = 10, cc_minor = 0;
  int l2_bytes = 126 << 20;
};
const DeviceProps &device_props(int dev);

extern uint64_t g_launches;  // atomic-incremented launch counter
void count_launch(uint64_t n = 1);

// ---- kernel launchers (return 0 or error code; set_error on failure) -----
int launch_vector_add(cudaStream_t s, int dev, uint64_t cov, const float *x,
                      const float *y, float *out);
int launch_saxpy(cudaStream_t s, int dev, uint64_t cov, float a, const float *x,
                 const float *y, float *out);
int launch_fill(cudaStream_t s, int dev, uint64_t cov, float v, float *out);
int launch_reduce_sum(cudaStream_t s, int dev, uint64_t n, const float *x, float *out);
// bt_prep: executor-owned buffer for B transposed ([m][k] f32) or nullptr;
// bt_ready: it already holds that (else it is filled first)
int launch_matmul(cudaStream_t s, int dev, uint64_t n, uint64_t m, uint64_t k, uint64_t cov,
                  const float *a, const float *b, float *out, StreamScratch *sc,
                  const float *bt_prep = nullptr, bool bt_ready = false);
int launch_jacobi(cudaStream_t s, int dev, int n, uint64_t cov, const float *A,
                  const float *b, const float *x_in, float *x_out, float *resid,
                  StreamScratch *sc);
// `sweeps` consecutive sweeps ping-ponging between x buffers, see jacobi.cu
struct JacobiChain {
  int n;
  uint64_t cov;
  const float *A;
  const float *b;
  int sweeps;
  const float *const *x_in;  // [sweeps]
  float *const *x_out;       // [sweeps]
  float *const *resid;       // [sweeps]
  // host (pinned, device-accessible) destinations the on-chip kernel writes
  // the LAST sweep's x_out / resid to as well (nullptr: none); *wb_done is
  // set when the chosen kernel did (otherwise the caller copies)
  float *wb_x = nullptr, *wb_r = nullptr;
  bool *wb_done = nullptr;
};
int launch_jacobi_chain(cudaStream_t s, int dev, const JacobiChain &c, StreamScratch *sc,
                        uint64_t memo_key = 0);
// relaunch the memoised chain of sc with these write-back destinations
// (returns 1 when there is none to relaunch)
int launch_jacobi_memo(cudaStream_t s, int dev, StreamScratch *sc, float *wb_x = nullptr, float *wb_r = nullptr);
void free_jacobi_memo(StreamScratch *sc);
// Prepared-operand buffers for cGEMM (nullptr = use per-stream scratch).
struct CgemmPrepared {
  float *a = nullptr;  // [A_hi; A_lo] fp16 + row max-bits
  float *b = nullptr;  // [Bt_hi; Bt_lo] fp16 + column max-bits
  bool a_ready = false, b_ready = false;
};
// fp16 elements per prepared operand row: 2k rounded up to 64 (128 bytes)
inline uint64_t cgemm_ldk16(uint64_t k) { return (2 * k + 63) / 64 * 64; }
// bytes of a prepared operand: side 0 = A (n rows), 1 = B (2m rows): hi and
// lo planes of fp16 rows, then 4 bytes of max-bits per row of A / complex
// column of B (gpu_executor.py computes the same sizes)
inline uint64_t cgemm_prepared_bytes(int side, uint64_t n, uint64_t m, uint64_t k) {
  const uint64_t ldk = cgemm_ldk16(k);
  return side == 0 ? 2 * n * ldk * 2 + 4 * n : 2 * (2 * m) * ldk * 2 + 4 * m;
}
int launch_cgemm(cudaStream_t s, int dev, int n, int m, int k, uint64_t cov,
                 const float *A, const float *B, float *C, StreamScratch *sc,
                 const ProgressiveOut *po = nullptr, const CgemmPrepared *prep = nullptr);

// ---- invocation runs (runs.cu): consecutive builtin invocations of one
// batch executed by one persistent cooperative launch
struct RunInv {
  int kernel;     // KAAS_K_*
  int flags;      // kaas_launch_desc.flags
  uint64_t ext[3];
  uint64_t cov;
  float fval;
  uint64_t ptr[4];
  uint64_t size[4];
};
bool run_eligible(const RunInv &v);
int launch_builtin_run(cudaStream_t s, int dev, StreamScratch *sc, const RunInv *v, int n);

}  // namespace kaas
