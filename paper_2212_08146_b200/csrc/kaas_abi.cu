// C-ABI layer of libkaas_b200.so: device/stream/event/memory/copy plumbing
// and the kernel dispatcher that stands in for SimulatedBackend.launch
// (pkg/src/kaas/backend.py:258-266).  See include/kaas_b200.h.
#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "kaas_internal.cuh"

namespace kaas {

// ---------------------------------------------------------------------------
// errors

static thread_local std::string t_last_error;

void set_error(const std::string &msg) { t_last_error = msg; }

int fail(int code, const std::string &msg) {
  set_error(msg);
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
  set_error(buf);
  return (int)e;
}

// ---------------------------------------------------------------------------
// device properties, scratch, counters

static std::mutex g_mu;
static std::unordered_map<int, DeviceProps> g_props;
static std::unordered_map<cudaStream_t, StreamScratch *> g_scratch;
static std::unordered_map<int, cudaEvent_t> g_coop_event;  // serialises cooperative grids per device
static std::atomic<uint64_t> g_launch_count{0};

void count_launch(uint64_t n) { g_launch_count.fetch_add(n, std::memory_order_relaxed); }

const DeviceProps &device_props(int dev) {
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_props.find(dev);
  if (it != g_props.end()) return it->second;
  DeviceProps p;
  cudaDeviceGetAttribute(&p.sm_count, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&p.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&p.cc_major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&p.cc_minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(&p.l2_bytes, cudaDevAttrL2CacheSize, dev);
  return g_props.emplace(dev, p).first->second;
}

StreamScratch *scratch_for(cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_scratch.find(s);
  return it == g_scratch.end() ? nullptr : it->second;
}

int ensure_matmul_scratch(StreamScratch *sc, cudaStream_t s, size_t bytes) {
  if (sc->mm_bytes >= bytes) return 0;
  if (sc->mm_buf) KAAS_CUDA(cudaFreeAsync(sc->mm_buf, s));
  sc->mm_buf = nullptr;
  sc->mm_bytes = 0;
  KAAS_CUDA(cudaMallocAsync(&sc->mm_buf, bytes, s));
  sc->mm_bytes = bytes;
  return 0;
}

int ensure_cgemm_scratch(StreamScratch *sc, cudaStream_t s, size_t bytes) {
  if (sc->cg_bytes >= bytes) return 0;
  if (sc->cg_buf) KAAS_CUDA(cudaFreeAsync(sc->cg_buf, s));
  sc->cg_buf = nullptr;
  sc->cg_bytes = 0;
  KAAS_CUDA(cudaMallocAsync(&sc->cg_buf, bytes, s));
  sc->cg_bytes = bytes;
  return 0;
}

static int stream_device(cudaStream_t s, int *dev) {
  StreamScratch *sc = scratch_for(s);
  if (!sc) return fail(KAAS_E_INVALID, "stream was not created by kaas_stream_create");
  *dev = sc->dev;
  return 0;
}

// Make the calling thread's current device the one `stream` belongs to, so
// every export works from any thread (a pool's worker threads, or a caller
// that drives an idle executor inline) whatever device it last touched.
static int bind_stream_device(cudaStream_t s) {
  int dev = 0, cur = -1;
  KAAS_CUDA(cudaStreamGetDevice(s, &dev));
  KAAS_CUDA(cudaGetDevice(&cur));
  if (cur != dev) KAAS_CUDA(cudaSetDevice(dev));
  return 0;
}

__global__ void k_inject_fault() { __trap(); }

// ---------------------------------------------------------------------------
// kernel table: literal signature, buffer count, written args
// (mirrors backend.py:236-243 plus the two new kernels)

struct KernelSig {
  int id;
  const char *name;
  int n_lits;
  int lit_tags[3];
  int n_args;
};

static const KernelSig kSigs[] = {
    {KAAS_K_VECTOR_ADD, "vector_add", 1, {KAAS_LIT_I32}, 3},
    {KAAS_K_SAXPY, "saxpy", 2, {KAAS_LIT_I32, KAAS_LIT_F32}, 3},
    {KAAS_K_MATMUL, "matmul", 3, {KAAS_LIT_I32, KAAS_LIT_I32, KAAS_LIT_I32}, 3},
    {KAAS_K_REDUCE_SUM, "reduce_sum", 1, {KAAS_LIT_I32}, 2},
    {KAAS_K_FILL, "fill", 2, {KAAS_LIT_I32, KAAS_LIT_F32}, 1},
    {KAAS_K_CGEMM, "cgemm", 3, {KAAS_LIT_I32, KAAS_LIT_I32, KAAS_LIT_I32}, 3},
    {KAAS_K_JACOBI, "jacobi_sweep", 1, {KAAS_LIT_I32}, 5},
};

static const KernelSig *find_sig(int id) {
  for (const auto &s : kSigs)
    if (s.id == id) return &s;
  return nullptr;
}

// A checked launch: extents, coverage and byte requirements resolved.
struct Plan {
  const KernelSig *sig;
  uint64_t ext[3];  // literal extents
  uint64_t cov;
  float fval;       // f32 literal (saxpy a / fill v), rounded once (backend.py:165,207)
};

static bool mul_ok(uint64_t a, uint64_t b, uint64_t *out) {
  if (a != 0 && b > UINT64_MAX / a) return false;
  *out = a * b;
  return true;
}

// _extent / _f32_view rules (backend.py:137-150), checked in the order the
// reference kernels evaluate them.
static int plan_launch(const kaas_launch_desc *d, Plan *p) {
  const KernelSig *sig = find_sig(d->kernel);
  if (!sig) return fail(KAAS_E_UNKNOWN_KERNEL, "unknown kernel id " + std::to_string(d->kernel));
  p->sig = sig;
  if (d->n_args != sig->n_args)
    return fail(KAAS_E_ARITY, std::string(sig->name) + ": expected " +
                                  std::to_string(sig->n_args) + " buffer args");
  if (d->n_lits != sig->n_lits) return fail(KAAS_E_ARITY, std::string(sig->name) + ": literal count");
  for (int i = 0; i < sig->n_lits; ++i)
    if (d->lits[i].tag != sig->lit_tags[i])
      return fail(KAAS_E_ARITY, std::string(sig->name) + ": literal types");
  uint64_t total = 1;
  for (int i = 0; i < 6; ++i) {
    if (d->dims[i] == 0) return fail(KAAS_E_INVALID, "launch dims must be >= 1");
    if (!mul_ok(total, d->dims[i], &total)) total = UINT64_MAX;
  }
  const int n_ext = (d->kernel == KAAS_K_MATMUL || d->kernel == KAAS_K_CGEMM) ? 3 : 1;
  for (int i = 0; i < n_ext; ++i) {
    if (d->lits[i].i < 0)
      return fail(KAAS_E_BOUNDS, std::string(sig->name) + ": extent must be non-negative");
    p->ext[i] = (uint64_t)d->lits[i].i;
  }
  p->fval = (sig->n_lits >= 2 && d->lits[1].tag == KAAS_LIT_F32) ? (float)d->lits[1].f : 0.0f;

  auto need = [&](int arg, uint64_t count, uint64_t elt) -> int {
    uint64_t bytes;
    if (!mul_ok(count, elt, &bytes) || bytes > d->sizes[arg])
      return fail(KAAS_E_BOUNDS, std::string(sig->name) + ": arg " + std::to_string(arg) +
                                     " needs more bytes than the buffer holds");
    return 0;
  };
  const uint64_t n = p->ext[0];
  int rc = 0;
  switch (d->kernel) {
    case KAAS_K_VECTOR_ADD:
    case KAAS_K_SAXPY:
      if ((rc = need(0, n, 4)) || (rc = need(1, n, 4)) || (rc = need(2, n, 4))) return rc;
      p->cov = total < n ? total : n;
      break;
    case KAAS_K_FILL:
      if ((rc = need(0, n, 4))) return rc;
      p->cov = total < n ? total : n;
      break;
    case KAAS_K_REDUCE_SUM:
      if ((rc = need(0, n, 4)) || (rc = need(1, 1, 4))) return rc;
      p->cov = n;
      break;
    case KAAS_K_MATMUL:
    case KAAS_K_CGEMM: {
      const uint64_t m = p->ext[1], k = p->ext[2];
      const uint64_t elt = d->kernel == KAAS_K_MATMUL ? 4 : 8;
      uint64_t nk, km, nm;
      if (!mul_ok(n, k, &nk) || !mul_ok(k, m, &km) || !mul_ok(n, m, &nm))
        return fail(KAAS_E_BOUNDS, std::string(sig->name) + ": extents overflow");
      if ((rc = need(0, nk, elt)) || (rc = need(1, km, elt)) || (rc = need(2, nm, elt))) return rc;
      p->cov = total < nm ? total : nm;
      break;
    }
    case KAAS_K_JACOBI: {
      uint64_t nn;
      if (!mul_ok(n, n, &nn)) return fail(KAAS_E_BOUNDS, "jacobi_sweep: extent overflow");
      if ((rc = need(0, nn, 4)) || (rc = need(1, n, 4)) || (rc = need(2, n, 4)) ||
          (rc = need(3, n, 4)) || (rc = need(4, 1, 4)))
        return rc;
      if (n > 0x7fffffff) return fail(KAAS_E_BOUNDS, "jacobi_sweep: n exceeds i32");
      p->cov = total < n ? total : n;
      break;
    }
  }
  return 0;
}

// Kernels that read some operand after writing another need the written
// operand redirected when the request binds one buffer to both (the
// reference reads every input before writing, backend.py:8-9).
static bool alias_unsafe(int kernel) {
  return kernel == KAAS_K_MATMUL || kernel == KAAS_K_CGEMM || kernel == KAAS_K_JACOBI;
}

static int written_args(int kernel, int *w) {
  switch (kernel) {
    case KAAS_K_FILL: w[0] = 0; return 1;
    case KAAS_K_REDUCE_SUM: w[0] = 1; return 1;
    case KAAS_K_JACOBI: w[0] = 3; w[1] = 4; return 2;
    default: w[0] = 2; return 1;
  }
}

static int run_plan(int dev, cudaStream_t s, const kaas_launch_desc *d, const Plan &p,
                    StreamScratch *sc, const ProgressiveOut *po = nullptr) {
  uint64_t ptr[KAAS_MAX_ARGS];
  memcpy(ptr, d->ptrs, sizeof ptr);

  // Alias redirection: a written arg that shares its buffer with a read arg
  // goes through a temporary holding a copy of the buffer (so the uncovered
  // tail survives), then is copied back.
  struct Redirect { uint64_t orig, tmp, bytes; };
  std::vector<Redirect> redirects;
  if (alias_unsafe(d->kernel)) {
    int w[2];
    const int nw = written_args(d->kernel, w);
    for (int wi = 0; wi < nw; ++wi) {
      const uint64_t target = d->ptrs[w[wi]];
      bool aliased = false;
      for (int a = 0; a < d->n_args; ++a) {
        bool is_written = false;
        for (int wj = 0; wj < nw; ++wj) is_written |= (w[wj] == a);
        if (!is_written && d->ptrs[a] == target) aliased = true;
      }
      if (!aliased) continue;
      bool have = false;
      for (auto &r : redirects) have |= (r.orig == target);
      if (have) continue;
      void *tmp = nullptr;
      KAAS_CUDA(cudaMallocAsync(&tmp, d->sizes[w[wi]], s));
      KAAS_CUDA(cudaMemcpyAsync(tmp, (void *)target, d->sizes[w[wi]], cudaMemcpyDeviceToDevice, s));
      redirects.push_back({target, (uint64_t)tmp, d->sizes[w[wi]]});
    }
    for (int wi = 0; wi < nw; ++wi)
      for (auto &r : redirects)
        if (d->ptrs[w[wi]] == r.orig) ptr[w[wi]] = r.tmp;
  }

  int rc = 0;
  const uint64_t n = p.ext[0];
  switch (d->kernel) {
    case KAAS_K_VECTOR_ADD:
      rc = launch_vector_add(s, dev, p.cov, (const float *)ptr[0], (const float *)ptr[1], (float *)ptr[2]);
      break;
    case KAAS_K_SAXPY:
      rc = launch_saxpy(s, dev, p.cov, p.fval, (const float *)ptr[0], (const float *)ptr[1], (float *)ptr[2]);
      break;
    case KAAS_K_FILL:
      rc = launch_fill(s, dev, p.cov, p.fval, (float *)ptr[0]);
      break;
    case KAAS_K_REDUCE_SUM:
      rc = launch_reduce_sum(s, dev, n, (const float *)ptr[0], (float *)ptr[1]);
      break;
    case KAAS_K_MATMUL: {
      const float *bt = nullptr;
      bool bt_ready = false;
      if (d->flags & (KAAS_F_MM_BT_USE | KAAS_F_MM_BT_FILL)) {
        if (d->sizes[3] < p.ext[1] * p.ext[2] * 4) return fail(KAAS_E_BOUNDS, "matmul: prepared B buffer too small");
        bt = (const float *)d->ptrs[3];
        bt_ready = (d->flags & KAAS_F_MM_BT_USE) != 0;
      }
      rc = launch_matmul(s, dev, n, p.ext[1], p.ext[2], p.cov, (const float *)ptr[0],
                         (const float *)ptr[1], (float *)ptr[2], sc, bt, bt_ready);
      break;
    }
    case KAAS_K_CGEMM: {
      if (n > 0x7fffffff || p.ext[1] > 0x7fffffff || p.ext[2] > 0x7fffffff)
        return fail(KAAS_E_BOUNDS, "cgemm: extent exceeds i32");
      CgemmPrepared prep;
      if (d->flags & (KAAS_F_CG_A_USE | KAAS_F_CG_A_FILL)) {
        if (d->sizes[3] < cgemm_prepared_bytes(0, n, p.ext[1], p.ext[2]))
          return fail(KAAS_E_BOUNDS, "cgemm: prepared A buffer too small");
        prep.a = (float *)d->ptrs[3];
        prep.a_ready = (d->flags & KAAS_F_CG_A_USE) != 0;
      }
      if (d->flags & (KAAS_F_CG_B_USE | KAAS_F_CG_B_FILL)) {
        if (d->sizes[4] < cgemm_prepared_bytes(1, n, p.ext[1], p.ext[2]))
          return fail(KAAS_E_BOUNDS, "cgemm: prepared B buffer too small");
        prep.b = (float *)d->ptrs[4];
        prep.b_ready = (d->flags & KAAS_F_CG_B_USE) != 0;
      }
      rc = launch_cgemm(s, dev, (int)n, (int)p.ext[1], (int)p.ext[2], p.cov, (const float *)ptr[0],
                        (const float *)ptr[1], (float *)ptr[2], sc,
                        (po && redirects.empty()) ? po : nullptr, &prep);
      break;
    }
      break;
    case KAAS_K_JACOBI:
      if (n == 0 || p.cov == 0) {
        // nothing covered: residual of an empty sum
        rc = launch_fill(s, dev, 1, 0.0f, (float *)ptr[4]);
        break;
      }
      rc = launch_jacobi(s, dev, (int)n, p.cov, (const float *)ptr[0], (const float *)ptr[1],
                         (const float *)ptr[2], (float *)ptr[3], (float *)ptr[4], sc);
      break;
  }
  if (rc) return rc;
  for (auto &r : redirects) {
    KAAS_CUDA(cudaMemcpyAsync((void *)r.orig, (void *)r.tmp, r.bytes, cudaMemcpyDeviceToDevice, s));
    KAAS_CUDA(cudaFreeAsync((void *)r.tmp, s));
  }
  if (po && !redirects.empty()) {  // aliased output went through a temporary: copy it whole
    cudaEvent_t ev;
    KAAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    KAAS_CUDA(cudaEventRecord(ev, s));
    KAAS_CUDA(cudaStreamWaitEvent(po->out_stream, ev, 0));
    KAAS_CUDA(cudaMemcpyAsync(po->host, (const void *)d->ptrs[2], po->bytes, cudaMemcpyDeviceToHost,
                              po->out_stream));
    cudaEventDestroy(ev);
  }
  return 0;
}

// A run of Jacobi sweeps that can share one persistent launch: same system,
// no buffer both read and written within a sweep, and residual slots that
// nothing in the run reads.
static int jacobi_run_length(const kaas_launch_desc *d, const Plan *plans, int i, int n) {
  const kaas_launch_desc &h = d[i];
  if (h.kernel != KAAS_K_JACOBI || plans[i].cov == 0) return 1;
  int j = i;
  for (; j < n; ++j) {
    const kaas_launch_desc &e = d[j];
    if (e.kernel != KAAS_K_JACOBI || plans[j].ext[0] != plans[i].ext[0] ||
        plans[j].cov != plans[i].cov || e.ptrs[0] != h.ptrs[0] || e.ptrs[1] != h.ptrs[1])
      break;
    const uint64_t A = e.ptrs[0], b = e.ptrs[1], xi = e.ptrs[2], xo = e.ptrs[3], r = e.ptrs[4];
    if (xo == xi || xo == A || xo == b || r == A || r == b || r == xi || r == xo) break;
  }
  // residual slots must not be read (as x_in) or written (as x_out) by any
  // sweep of the run: the run ends before the first sweep that conflicts
  // with itself or an earlier one.  A run touches only a handful of distinct
  // buffers, so the seen-sets are short vectors (linear in the run length;
  // the all-pairs check cost ~140 us of host time per 500-sweep request).
  std::vector<uint64_t> xs, rs;
  auto has = [](const std::vector<uint64_t> &v, uint64_t q) {
    for (uint64_t e : v)
      if (e == q) return true;
    return false;
  };
  auto add = [&](std::vector<uint64_t> &v, uint64_t q) {
    if (!has(v, q)) v.push_back(q);
  };
  int len = j - i;
  for (int t = i; t < i + len; ++t) {
    const uint64_t xi = d[t].ptrs[2], xo = d[t].ptrs[3], r = d[t].ptrs[4];
    add(xs, xi);
    add(xs, xo);
    if (has(xs, r) || has(rs, xi) || has(rs, xo)) {
      len = t - i;
      break;
    }
    add(rs, r);
  }
  return len < 1 ? 1 : len;
}

// invocation runs: the shortest run worth one persistent launch, and the dev
// A/B switch (KAAS_RUN=0: every invocation launches on its own)
constexpr int kRunMinLength = 2;
static bool run_use_enabled() {
  const char *e = KAAS_DEV_ENV("KAAS_RUN");
  return !(e && e[0] == '0');
}

// Cooperative grids on one device must not overlap (two persistent grids
// that each need every SM could wait on each other forever).  Launches on
// one stream are ordered already; when the next cooperative launch comes
// from a different stream than the last one, it first waits for everything
// enqueued so far on that stream.  The per-device mutex is held from
// coop_serialise_begin to coop_serialise_end, so check, launch and hand-over
// are one step even with several executor threads on a device.
static std::mutex g_coop_mu;
static std::unordered_map<int, cudaStream_t> g_coop_last;  // last stream with a cooperative grid, per device

static int coop_serialise_begin(int dev, cudaStream_t s) {
  g_coop_mu.lock();
  auto last = g_coop_last.find(dev);
  if (last == g_coop_last.end() || last->second == s) return 0;
  auto it = g_coop_event.find(dev);
  if (it == g_coop_event.end()) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      g_coop_mu.unlock();
      return cuda_fail(e, "cudaEventCreateWithFlags");
    }
    it = g_coop_event.emplace(dev, ev).first;
  }
  cudaError_t e = cudaEventRecord(it->second, last->second);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, it->second, 0);
  if (e != cudaSuccess) {
    g_coop_mu.unlock();
    return cuda_fail(e, "cooperative hand-over");
  }
  return 0;
}

// rc: the launch's result; always releases the mutex taken by _begin
static int coop_serialise_end(int dev, cudaStream_t s, int rc = 0) {
  if (rc == 0) g_coop_last[dev] = s;
  g_coop_mu.unlock();
  return rc;
}

}  // namespace kaas

using namespace kaas;

// ===========================================================================
// exported C ABI

extern "C" {

int kaas_last_error(char *buf, size_t len) {
  if (!buf || len == 0) return KAAS_E_INVALID;
  snprintf(buf, len, "%s", t_last_error.c_str());
  return 0;
}

int kaas_version(int *major, int *minor) {
  if (major) *major = 1;
  if (minor) *minor = 0;
  return 0;
}

int kaas_device_count(int *n) {
  if (!n) return KAAS_E_INVALID;
  cudaError_t e = cudaGetDeviceCount(n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    cudaGetLastError();
    *n = 0;
    return 0;
  }
  KAAS_CUDA(e);
  return 0;
}

int kaas_init_device(int dev) {
  KAAS_CUDA(cudaSetDevice(dev));
  const DeviceProps &p = device_props(dev);
  if (p.cc_major != 10)
    return fail(KAAS_E_UNSUPPORTED, "libkaas_b200 is built for sm_100a; device " +
                                        std::to_string(dev) + " is sm_" + std::to_string(p.cc_major) +
                                        std::to_string(p.cc_minor));
  cudaMemPool_t pool;
  KAAS_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;  // never hand pages back to the OS between requests
  KAAS_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  KAAS_CUDA(cudaFree(nullptr));
  return 0;
}

int kaas_device_info_get(int dev, kaas_device_info *out) {
  if (!out) return KAAS_E_INVALID;
  cudaDeviceProp prop;
  KAAS_CUDA(cudaGetDeviceProperties(&prop, dev));
  memset(out, 0, sizeof *out);
  out->ordinal = dev;
  out->sm_count = prop.multiProcessorCount;
  out->cc_major = prop.major;
  out->cc_minor = prop.minor;
  out->total_mem = prop.totalGlobalMem;
  out->l2_bytes = (uint64_t)prop.l2CacheSize;
  out->max_smem_per_block = (int)prop.sharedMemPerBlockOptin;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  out->clock_khz = clk;
  snprintf(out->name, sizeof out->name, "%s", prop.name);
  return 0;
}

int kaas_launch_counter(uint64_t *out) {
  if (!out) return KAAS_E_INVALID;
  *out = g_launch_count.load();
  return 0;
}

// ---- streams / events ------------------------------------------------------

int kaas_stream_create(int dev, int priority, uint64_t *stream) {
  if (!stream) return KAAS_E_INVALID;
  KAAS_CUDA(cudaSetDevice(dev));
  cudaStream_t s;
  KAAS_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority));
  auto *sc = new StreamScratch();
  sc->dev = dev;
  cudaError_t e = cudaMallocAsync((void **)&sc->jac_partials, 2 * kMaxJacobiBlocks * sizeof(float), s);
  if (e == cudaSuccess) e = cudaMallocAsync((void **)&sc->jac_sync, 16 * sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(sc->jac_sync, 0, 16 * sizeof(unsigned), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync((void **)&sc->jac_xt, 2 * kJacTaggedMaxN * sizeof(unsigned long long), s);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(sc->jac_xt, 0, 2 * kJacTaggedMaxN * sizeof(unsigned long long), s);
  // stream memory operations (cuStreamWaitValue32) target plain device memory
  if (e == cudaSuccess) e = cudaMalloc((void **)&sc->panel_done, kMaxPanels * sizeof(unsigned));
  if (e != cudaSuccess) {
    delete sc;
    cudaStreamDestroy(s);
    return cuda_fail(e, "stream scratch allocation");
  }
  {
    std::lock_guard<std::mutex> g(g_mu);
    g_scratch[s] = sc;
  }
  *stream = (uint64_t)s;
  return 0;
}

int kaas_stream_destroy(uint64_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  StreamScratch *sc = nullptr;
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_scratch.find(s);
    if (it != g_scratch.end()) {
      sc = it->second;
      g_scratch.erase(it);
    }
  }
  if (sc) {
    cudaSetDevice(sc->dev);
    if (sc->jac_partials) cudaFreeAsync(sc->jac_partials, s);
    if (sc->jac_sync) cudaFreeAsync(sc->jac_sync, s);
    if (sc->jac_xt) cudaFreeAsync(sc->jac_xt, s);
    if (sc->cg_buf) cudaFreeAsync(sc->cg_buf, s);
    free_jacobi_memo(sc);
    if (sc->mm_buf) cudaFreeAsync(sc->mm_buf, s);
    if (sc->run_done) cudaFreeAsync(sc->run_done, s);
    cudaStreamSynchronize(s);
    {
      // its grids are finished: a later cooperative launch from another
      // stream must not hand over from this one once it is destroyed
      std::lock_guard<std::mutex> g(g_coop_mu);
      for (auto it = g_coop_last.begin(); it != g_coop_last.end();)
        it = it->second == s ? g_coop_last.erase(it) : std::next(it);
    }
    if (sc->panel_done) cudaFree(sc->panel_done);
    if (sc->cg_ev_ready) cudaEventDestroy(sc->cg_ev_ready);
    if (sc->cg_ev_done) cudaEventDestroy(sc->cg_ev_done);
    delete sc;
  }
  KAAS_CUDA(cudaStreamDestroy(s));
  return 0;
}

int kaas_stream_sync(uint64_t stream) {
  KAAS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return 0;
}

int kaas_event_create(int dev, int timing, uint64_t *event) {
  if (!event) return KAAS_E_INVALID;
  KAAS_CUDA(cudaSetDevice(dev));
  cudaEvent_t e;
  KAAS_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *event = (uint64_t)e;
  return 0;
}

int kaas_event_destroy(uint64_t event) {
  KAAS_CUDA(cudaEventDestroy((cudaEvent_t)event));
  return 0;
}

int kaas_event_record(uint64_t event, uint64_t stream) {
  KAAS_CUDA(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
  return 0;
}

int kaas_stream_wait_event(uint64_t stream, uint64_t event) {
  KAAS_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
  return 0;
}

int kaas_event_sync(uint64_t event) {
  KAAS_CUDA(cudaEventSynchronize((cudaEvent_t)event));
  return 0;
}

int kaas_event_query(uint64_t event, int *done) {
  if (!done) return KAAS_E_INVALID;
  cudaError_t e = cudaEventQuery((cudaEvent_t)event);
  if (e == cudaErrorNotReady) {
    *done = 0;
    return 0;
  }
  KAAS_CUDA(e);
  *done = 1;
  return 0;
}

int kaas_event_elapsed_ms(uint64_t start, uint64_t end, float *ms) {
  if (!ms) return KAAS_E_INVALID;
  KAAS_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)end));
  return 0;
}

int kaas_event_elapsed_many(int n, const uint64_t *starts, const uint64_t *ends, float *ms) {
  if (n < 0 || (n > 0 && (!starts || !ends || !ms))) return KAAS_E_INVALID;
  for (int i = 0; i < n; ++i)
    KAAS_CUDA(cudaEventElapsedTime(&ms[i], (cudaEvent_t)starts[i], (cudaEvent_t)ends[i]));
  return 0;
}

// ---- memory ----------------------------------------------------------------

int kaas_malloc_async(uint64_t stream, uint64_t bytes, uint64_t *dptr) {
  if (!dptr) return KAAS_E_INVALID;
  int dev, rc;
  if ((rc = stream_device((cudaStream_t)stream, &dev))) return rc;
  KAAS_CUDA(cudaSetDevice(dev));
  void *p = nullptr;
  KAAS_CUDA(cudaMallocAsync(&p, bytes ? bytes : 1, (cudaStream_t)stream));
  *dptr = (uint64_t)p;
  return 0;
}

int kaas_free_async(uint64_t stream, uint64_t dptr) {
  int dev, rc;
  if ((rc = stream_device((cudaStream_t)stream, &dev))) return rc;
  KAAS_CUDA(cudaSetDevice(dev));
  KAAS_CUDA(cudaFreeAsync((void *)dptr, (cudaStream_t)stream));
  return 0;
}

int kaas_memset_async(uint64_t dptr, int value, uint64_t bytes, uint64_t stream) {
  if (bytes == 0) return 0;
  if (int rc = bind_stream_device((cudaStream_t)stream)) return rc;
  KAAS_CUDA(cudaMemsetAsync((void *)dptr, value, bytes, (cudaStream_t)stream));
  return 0;
}

int kaas_host_alloc(uint64_t bytes, void **ptr) {
  if (!ptr) return KAAS_E_INVALID;
  KAAS_CUDA(cudaHostAlloc(ptr, bytes ? bytes : 1, cudaHostAllocPortable));
  return 0;
}

int kaas_host_free(void *ptr) {
  KAAS_CUDA(cudaFreeHost(ptr));
  return 0;
}

int kaas_host_register(void *ptr, uint64_t bytes) {
  KAAS_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterPortable));
  return 0;
}

int kaas_host_unregister(void *ptr) {
  KAAS_CUDA(cudaHostUnregister(ptr));
  return 0;
}

// ---- copies ----------------------------------------------------------------

int kaas_memcpy_h2d_async(uint64_t dst, const void *src, uint64_t bytes, uint64_t stream) {
  if (bytes == 0) return 0;
  if (int rc = bind_stream_device((cudaStream_t)stream)) return rc;
  KAAS_CUDA(cudaMemcpyAsync((void *)dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return 0;
}

int kaas_memcpy_d2h_async(void *dst, uint64_t src, uint64_t bytes, uint64_t stream) {
  if (bytes == 0) return 0;
  if (int rc = bind_stream_device((cudaStream_t)stream)) return rc;
  KAAS_CUDA(cudaMemcpyAsync(dst, (const void *)src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return 0;
}

int kaas_memcpy_d2d_async(uint64_t dst, uint64_t src, uint64_t bytes, uint64_t stream) {
  if (bytes == 0) return 0;
  if (int rc = bind_stream_device((cudaStream_t)stream)) return rc;
  KAAS_CUDA(cudaMemcpyAsync((void *)dst, (const void *)src, bytes, cudaMemcpyDeviceToDevice,
                            (cudaStream_t)stream));
  return 0;
}

int kaas_enable_peer(int dev, int peer) {
  KAAS_CUDA(cudaSetDevice(dev));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
  } else {
    KAAS_CUDA(e);
  }
  // Cache entries come from the peer's stream-ordered pool: peer access to
  // pool memory is granted per pool (cudaDeviceEnablePeerAccess covers only
  // cudaMalloc memory), so let `dev` map `peer`'s pool allocations too.
  if (dev != peer) {
    cudaMemPool_t pool;
    KAAS_CUDA(cudaDeviceGetDefaultMemPool(&pool, peer));
    cudaMemAccessDesc desc = {};
    desc.location.type = cudaMemLocationTypeDevice;
    desc.location.id = dev;
    desc.flags = cudaMemAccessFlagsProtReadWrite;
    KAAS_CUDA(cudaMemPoolSetAccess(pool, &desc, 1));
  }
  return 0;
}

int kaas_device_check(int dev) {
  KAAS_CUDA(cudaSetDevice(dev));
  KAAS_CUDA(cudaDeviceSynchronize());  // a sticky fault reports here on every call
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

int kaas_inject_fault(uint64_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (int rc = bind_stream_device(s)) return rc;
  k_inject_fault<<<1, 1, 0, s>>>();
  count_launch();
  KAAS_CUDA(cudaGetLastError());
  return 0;
}

int kaas_can_access_peer(int dev, int peer, int *can) {
  if (!can) return KAAS_E_INVALID;
  KAAS_CUDA(cudaDeviceCanAccessPeer(can, dev, peer));
  return 0;
}

int kaas_memcpy_p2p_async(uint64_t dst, int dst_dev, uint64_t src, int src_dev, uint64_t bytes,
                          uint64_t stream) {
  if (bytes == 0) return 0;
  if (int rc = bind_stream_device((cudaStream_t)stream)) return rc;
  KAAS_CUDA(cudaMemcpyPeerAsync((void *)dst, dst_dev, (const void *)src, src_dev, bytes,
                                (cudaStream_t)stream));
  return 0;
}

// ---- kernels -----------------------------------------------------------------

int kaas_launch(int dev, uint64_t stream, const kaas_launch_desc *desc) {
  return kaas_launch_batch(dev, stream, desc, 1);
}

int kaas_launch_batch(int dev, uint64_t stream, const kaas_launch_desc *descs, int n) {
  return kaas_launch_batch_ex(dev, stream, descs, n, nullptr, 0);
}

static int launch_batch_impl(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                             const kaas_stream_out *outs, int n_outs, uint64_t memo_key);

int kaas_launch_batch_ex(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                         const kaas_stream_out *outs, int n_outs) {
  return launch_batch_impl(dev, stream, descs, n, outs, n_outs, 0);
}

int kaas_launch_batch_memo(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                           uint64_t memo_key) {
  if (memo_key) {
    StreamScratch *sc = scratch_for((cudaStream_t)stream);
    if (sc && sc->dev == dev && sc->jac_memo_key == memo_key && n > 0 && descs) {
      KAAS_CUDA(cudaSetDevice(dev));
      cudaStream_t s = (cudaStream_t)stream;
      int rc;
      if ((rc = coop_serialise_begin(dev, s))) return rc;
      rc = coop_serialise_end(dev, s, launch_jacobi_memo(s, dev, sc));
      if (rc == 0) return 0;
      if (rc != 1) return rc;  // 1: nothing memoised after all -- take the full path
    }
  }
  return launch_batch_impl(dev, stream, descs, n, nullptr, 0, memo_key);
}

int kaas_launch_batch_timed(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                            uint64_t memo_key, uint64_t join_stream, uint64_t join_event,
                            uint64_t ev_start, uint64_t ev_end, const kaas_stream_out *outs,
                            int n_outs) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n_outs < 0 || (n_outs > 0 && !outs)) return fail(KAAS_E_INVALID, "null stream-out specs");
  if (join_event) {
    KAAS_CUDA(cudaEventRecord((cudaEvent_t)join_event, (cudaStream_t)join_stream));
    KAAS_CUDA(cudaStreamWaitEvent(s, (cudaEvent_t)join_event, 0));
  }
  if (ev_start) KAAS_CUDA(cudaEventRecord((cudaEvent_t)ev_start, s));
  int rc = 1;
  if (memo_key && n > 0 && descs) {
    // a memoised Jacobi chain whose stream-outs are exactly its last sweep's
    // x_out / resid: relaunch it with those as its write-back destinations
    StreamScratch *sc = scratch_for(s);
    float *wb_x = nullptr, *wb_r = nullptr;
    bool ok = sc && sc->dev == dev && sc->jac_memo_key == memo_key && descs[n - 1].kernel == KAAS_K_JACOBI;
    for (int o = 0; o < n_outs && ok; ++o) {
      const kaas_stream_out &so = outs[o];
      // the kernel writes exactly x[0:n] (arg 3) / the one residual (arg 4)
      const uint64_t nx = 4 * (uint64_t)descs[n - 1].lits[0].i;
      ok = so.desc_index == n - 1 && so.host_dst &&
           ((so.arg_index == 3 && so.bytes == nx && descs[n - 1].sizes[3] == nx) ||
            (so.arg_index == 4 && so.bytes == 4 && descs[n - 1].sizes[4] == 4));
      if (ok) (so.arg_index == 3 ? wb_x : wb_r) = (float *)so.host_dst;
    }
    if (ok) {
      KAAS_CUDA(cudaSetDevice(dev));
      if ((rc = coop_serialise_begin(dev, s))) return rc;
      rc = coop_serialise_end(dev, s, launch_jacobi_memo(s, dev, sc, wb_x, wb_r));
      if (rc != 0 && rc != 1) return rc;
    }
  }
  if (rc == 1 && (rc = launch_batch_impl(dev, stream, descs, n, outs, n_outs, memo_key))) return rc;
  if (ev_end) KAAS_CUDA(cudaEventRecord((cudaEvent_t)ev_end, s));
  return 0;
}

static int launch_batch_impl(int dev, uint64_t stream, const kaas_launch_desc *descs, int n,
                             const kaas_stream_out *outs, int n_outs, uint64_t memo_key) {
  if (n < 0 || (n > 0 && !descs)) return fail(KAAS_E_INVALID, "null launch descriptors");
  if (n_outs < 0 || (n_outs > 0 && !outs)) return fail(KAAS_E_INVALID, "null stream-out specs");
  cudaStream_t s = (cudaStream_t)stream;
  StreamScratch *sc = scratch_for(s);
  if (!sc) return fail(KAAS_E_INVALID, "stream was not created by kaas_stream_create");
  if (sc->dev != dev) return fail(KAAS_E_INVALID, "stream belongs to another device");
  KAAS_CUDA(cudaSetDevice(dev));
  std::vector<Plan> plans((size_t)n);
  for (int i = 0; i < n; ++i) {
    // a plan depends on everything but the pointers: a run of identical
    // invocations (a Jacobi chain's 500 sweeps) is validated once
    if (i > 0 && std::memcmp(&descs[i], &descs[i - 1], offsetof(kaas_launch_desc, ptrs)) == 0 &&
        std::memcmp(descs[i].sizes, descs[i - 1].sizes, sizeof(descs[i].sizes)) == 0) {
      plans[i] = plans[i - 1];
      continue;
    }
    int rc = plan_launch(&descs[i], &plans[i]);
    if (rc) {
      set_error("invocation " + std::to_string(i) + ": " + t_last_error);
      return rc;
    }
  }
  // stream-out specs: validate, and pick the ones a kernel can stream itself
  std::vector<int> prog_of(n, -1);     // desc -> out spec streamed progressively
  std::vector<char> done_out(n_outs, 0);
  for (int o = 0; o < n_outs; ++o) {
    const kaas_stream_out &so = outs[o];
    if (so.desc_index < 0 || so.desc_index >= n || so.arg_index < 0 ||
        so.arg_index >= descs[so.desc_index].n_args || !so.host_dst ||
        so.bytes > descs[so.desc_index].sizes[so.arg_index])
      return fail(KAAS_E_INVALID, "bad stream-out spec");
    const uint64_t target = descs[so.desc_index].ptrs[so.arg_index];
    for (int j = so.desc_index + 1; j < n; ++j) {  // must be the last writer of the buffer
      int w[2];
      const int nw = written_args(descs[j].kernel, w);
      for (int q = 0; q < nw; ++q)
        if (descs[j].ptrs[w[q]] == target)
          return fail(KAAS_E_INVALID, "stream-out buffer is written again later in the batch");
    }
    if (descs[so.desc_index].kernel == KAAS_K_CGEMM && so.arg_index == 2) prog_of[so.desc_index] = o;
  }
  std::vector<const float *> xin, xout, res;
  for (int i = 0; i < n;) {
    const int run = jacobi_run_length(descs, plans.data(), i, n);
    if (run >= 2) {
      xin.resize(run);
      xout.resize(run);
      res.resize(run);
      for (int t = 0; t < run; ++t) {
        xin[t] = (const float *)descs[i + t].ptrs[2];
        xout[t] = (const float *)descs[i + t].ptrs[3];
        res[t] = (const float *)descs[i + t].ptrs[4];
      }
      JacobiChain c{(int)plans[i].ext[0], plans[i].cov, (const float *)descs[i].ptrs[0],
                    (const float *)descs[i].ptrs[1], run, xin.data(),
                    (float *const *)xout.data(), (float *const *)res.data()};
      // stream-outs of the run's last sweep's x_out / resid: written back by
      // the kernel itself when it can (else copied below)
      int wb_o[2] = {-1, -1};
      const uint64_t nx = 4 * (uint64_t)plans[i].ext[0];
      for (int o = 0; o < n_outs; ++o) {
        const kaas_stream_out &so = outs[o];
        const int last = i + run - 1;
        // the kernel writes exactly x[0:n] / the one residual
        if (!done_out[o] && so.desc_index == last &&
            ((so.arg_index == 3 && so.bytes == nx && descs[last].sizes[3] == nx) ||
             (so.arg_index == 4 && so.bytes == 4 && descs[last].sizes[4] == 4)))
          wb_o[so.arg_index - 3] = o;
      }
      bool wb_done = false;
      c.wb_x = wb_o[0] >= 0 ? (float *)outs[wb_o[0]].host_dst : nullptr;
      c.wb_r = wb_o[1] >= 0 ? (float *)outs[wb_o[1]].host_dst : nullptr;
      c.wb_done = &wb_done;
      int rc;
      if ((rc = coop_serialise_begin(dev, s))) return rc;
      // the whole batch is this one run: the caller's memo key may name it
      if ((rc = coop_serialise_end(dev, s, launch_jacobi_chain(s, dev, c, sc, (i == 0 && run == n) ? memo_key : 0))))
        return rc;
      if (wb_done)
        for (int q = 0; q < 2; ++q)
          if (wb_o[q] >= 0) done_out[wb_o[q]] = 1;
      i += run;
      continue;
    }
    // a run of >= 2 builtin invocations: one persistent launch (runs.cu)
    {
      auto inv_of = [&](int j) {
        RunInv r{};
        const kaas_launch_desc &d = descs[j];
        r.kernel = d.kernel;
        r.flags = d.flags;
        memcpy(r.ext, plans[j].ext, sizeof r.ext);
        r.cov = plans[j].cov;
        r.fval = plans[j].fval;
        for (int q = 0; q < 4; ++q) {
          r.ptr[q] = q < KAAS_MAX_ARGS ? d.ptrs[q] : 0;
          r.size[q] = q < KAAS_MAX_ARGS ? d.sizes[q] : 0;
        }
        return r;
      };
      int len = 0;
      while (i + len < n && run_use_enabled() && run_eligible(inv_of(i + len))) ++len;
      if (len >= kRunMinLength) {
        std::vector<RunInv> inv((size_t)len);
        for (int t = 0; t < len; ++t) inv[t] = inv_of(i + t);
        int rc;
        if ((rc = coop_serialise_begin(dev, s))) return rc;
        if ((rc = coop_serialise_end(dev, s, launch_builtin_run(s, dev, sc, inv.data(), len)))) return rc;
        i += len;
        continue;
      }
    }
    ProgressiveOut po;
    const ProgressiveOut *pop = nullptr;
    if (prog_of[i] >= 0) {
      const kaas_stream_out &so = outs[prog_of[i]];
      po = {(cudaStream_t)so.out_stream, so.host_dst, so.bytes};
      pop = &po;
      done_out[prog_of[i]] = 1;
    }
    int rc = run_plan(dev, s, &descs[i], plans[i], sc, pop);
    if (rc) return rc;
    ++i;
  }
  // remaining stream-outs: one copy each after the whole batch
  if (n_outs) {
    cudaEvent_t ev = nullptr;
    for (int o = 0; o < n_outs; ++o) {
      if (done_out[o]) continue;
      if (!ev) {
        KAAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        KAAS_CUDA(cudaEventRecord(ev, s));
      }
      const kaas_stream_out &so = outs[o];
      KAAS_CUDA(cudaStreamWaitEvent((cudaStream_t)so.out_stream, ev, 0));
      KAAS_CUDA(cudaMemcpyAsync(so.host_dst, (const void *)descs[so.desc_index].ptrs[so.arg_index],
                                so.bytes, cudaMemcpyDeviceToHost, (cudaStream_t)so.out_stream));
    }
    if (ev) cudaEventDestroy(ev);
  }
  return 0;
}

}  // extern "C"
