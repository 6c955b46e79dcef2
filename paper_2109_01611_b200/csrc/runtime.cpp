// libgpulet host runtime: the C-ABI of include/gpulet.h.
//
// gpu-lets (§2.3) are green contexts over disjoint 8-SM
// groups of one GPU (cuDevSmResourceSplitByCount, minimum 8 SMs on CC >= 9.0),
// each running one persistent executor kernel (executor.cu) that pulls batch
// descriptors from a host-mapped ring and pushes completion records back
// (SURVEY.md §8(a) a1, a6, a7, a13).  The paper's frontend/backend processes,
// Unix sockets and MPS daemon are replaced by this in-process ABI.
#include <cuda.h>
#include <cuda_runtime.h>
#include <time.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <deque>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gpulet.h"
#include "runtime.h"

extern "C" cudaKernel_t gl_executor_handle();
extern "C" cudaKernel_t gl_probe_handle();
extern "C" const void* gl_executor_fn();

namespace gl {

static thread_local std::string g_err = "";

static gl_status fail(gl_status s, const std::string& m) {
  g_err = m;
  return s;
}

// the same thread-local error text for the stand-alone stage kernels (detect.cu)
gl_status set_error(gl_status s, const char* m) { return fail(s, m); }

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fp) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPointByVersion(name, fp, 12080, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    bool ok = true;
    ok &= get("cuTensorMapEncodeTiled", (void**)&d.tensorMapEncodeTiled);
    ok &= get("cuTensorMapEncodeIm2col", (void**)&d.tensorMapEncodeIm2col);
    ok &= get("cuDeviceGetDevResource", (void**)&d.deviceGetDevResource);
    ok &= get("cuDevSmResourceSplitByCount", (void**)&d.devSmResourceSplitByCount);
    ok &= get("cuDevResourceGenerateDesc", (void**)&d.devResourceGenerateDesc);
    ok &= get("cuGreenCtxCreate", (void**)&d.greenCtxCreate);
    ok &= get("cuGreenCtxDestroy", (void**)&d.greenCtxDestroy);
    ok &= get("cuGreenCtxStreamCreate", (void**)&d.greenCtxStreamCreate);
    ok &= get("cuLaunchKernelEx", (void**)&d.launchKernelEx);
    ok &= get("cuKernelSetAttribute", (void**)&d.kernelSetAttribute);
    ok &= get("cuStreamDestroy", (void**)&d.streamDestroy);
    ok &= get("cuDeviceGet", (void**)&d.deviceGet);
    d.ok = ok;
  });
  return d;
}

// Device frees while any persistent executor runs would block (cudaFree
// synchronises the device); they are deferred until no executor is alive.
static std::mutex g_free_mu;
static std::vector<std::pair<void*, bool>> g_deferred;
static std::atomic<int> g_live_exec{0};

void release_device(void* p, bool host) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_free_mu);
  if (g_live_exec.load() == 0) {
    if (host)
      cudaFreeHost(p);
    else
      cudaFree(p);
  } else {
    g_deferred.push_back({p, host});
  }
}

static void flush_deferred() {
  std::lock_guard<std::mutex> lk(g_free_mu);
  if (g_live_exec.load() != 0) return;
  for (auto& d : g_deferred) {
    if (d.second)
      cudaFreeHost(d.first);
    else
      cudaFree(d.first);
  }
  g_deferred.clear();
}

// GL_DEBUG=1: progress messages on stderr (host-side hang diagnosis).
static void dbg_log(const char* what) {
  static const bool on = getenv("GL_DEBUG") != nullptr;
  if (on) {
    fprintf(stderr, "[libgpulet] %s\n", what);
    fflush(stderr);
  }
}

static uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + ts.tv_nsec;
}

// ------------------------------------------------------------------ weight files
bool load_glw(const std::string& path, ParamMap& out, std::string& err) {
  std::ifstream f(path, std::ios::binary);
  if (!f) {
    err = "cannot open " + path;
    return false;
  }
  std::string first;
  std::getline(f, first);
  size_t hdr = 0;
  if (sscanf(first.c_str(), "GLW1 %zu", &hdr) != 1 || hdr == 0) {
    err = "not a GLW1 file: " + path;
    return false;
  }
  struct Ent {
    std::string name;
    std::vector<int> shape;
    size_t off, nbytes;
  };
  std::vector<Ent> ents;
  std::string line;
  while (std::getline(f, line)) {
    if (line == "END") break;
    std::istringstream ss(line);
    Ent e;
    std::string dtype;
    int nd = 0;
    ss >> e.name >> dtype >> nd;
    if (!ss || dtype != "bf16" || nd < 1 || nd > 6) {
      err = "bad header line: " + line;
      return false;
    }
    e.shape.resize(nd);
    for (int i = 0; i < nd; ++i) ss >> e.shape[i];
    ss >> e.off >> e.nbytes;
    if (!ss) {
      err = "bad header line: " + line;
      return false;
    }
    ents.push_back(e);
  }
  for (auto& e : ents) {
    Param p;
    p.shape = e.shape;
    if (p.numel() * 2 != e.nbytes) {
      err = "size mismatch for " + e.name;
      return false;
    }
    p.data.resize(p.numel());
    f.seekg((std::streamoff)(hdr + e.off));
    f.read((char*)p.data.data(), (std::streamsize)e.nbytes);
    if (!f) {
      err = "truncated data for " + e.name;
      return false;
    }
    out[e.name] = std::move(p);
  }
  return true;
}

}  // namespace gl

using namespace gl;

// ------------------------------------------------------------------ context objects
struct Gpulet {
  int id = -1, gpu = 0, slot = 0, pct = 100, nsm = 0;
  bool alive = false;
  CUgreenCtx gctx = nullptr;
  CUstream stream = nullptr;
  bool own_primary_stream = false;
  HostRing* ring = nullptr;      // host view
  HostRing* ring_dev = nullptr;  // device alias
  ExecState* st = nullptr;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  int* smid = nullptr;
  uint64_t tail = 0;       // items published
  uint64_t comp_seen = 0;  // completions consumed by the host
  std::vector<int> groups;
  bool uses_rem = false;
  bool unconfined = false;  // primary context, no green context (F4 "MPS(default)" analogue)
};

// Upload a program bound to workspace `ws` (tensor maps of workspace operands).
// The program's completion counters (barrier-free GEMM step joins) follow its
// descriptors in the same allocation, zeroed here; the executor re-zeroes them
// at the end of every run of the program.
static OpDesc* upload_bound(const Program& p, char* ws, std::string& err) {
  std::vector<OpDesc> ops;
  if (!bind_program(p, ws, ops, err)) return nullptr;
  OpDesc* d = nullptr;
  const size_t ob = ops.size() * sizeof(OpDesc);
  const size_t cb = ops.empty() ? 0 : (size_t)ops[0].cnt_words * 4;
  if (cudaMalloc(&d, ob + cb) != cudaSuccess) {
    err = "cudaMalloc(program)";
    return nullptr;
  }
  if (cb) {
    ops[0].cnt_base = (uint64_t)(uintptr_t)((char*)d + ob);
    cudaMemset((char*)d + ob, 0, cb);
  }
  cudaMemcpy(d, ops.data(), ob, cudaMemcpyHostToDevice);
  return d;
}

// Resources of one gpu-let slot of a GPU, reused by successive gpu-lets.
struct SlotRes {
  bool ready = false;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  HostRing* ring = nullptr;
  HostRing* ring_dev = nullptr;
  ExecState* st = nullptr;
  int* smid = nullptr;
  std::map<int, std::vector<OpDesc*>> progs;  // model id -> [batch] programs bound to ws (148-SM tiling)
  // (model id, SM count) -> [batch] programs tiled for that gpu-let size, bound to ws
  std::map<std::pair<int, int>, std::vector<OpDesc*>> progs_sm;
};

constexpr int kMaxSlots = 4;   // gpu-lets per GPU: 2 by gl_create_gpulet, up to 4 by gl_create_gpulets

struct GpuState {
  SlotRes slot_res[kMaxSlots];
  bool green_ready = false;
  CUgreenCtx gctx[kMaxSlots][5] = {};      // [slot][size index of 20,40,50,60,80]
  CUstream gstream[kMaxSlots][5] = {};
  int gnsm[kMaxSlots][5] = {};
  CUstream full_stream = nullptr;  // 100 %: a non-blocking stream of the primary context
  CUstream ustream[kMaxSlots] = {};  // unconfined executors: one non-blocking primary stream per slot
  bool multi = false;              // a partition of 3-4 gpu-lets: slot s holds SM pairs from layout_pair[s] on
  int layout_pair[kMaxSlots] = {};
  int dev = 0;
  int nsm = 0;
  bool split = false;
  CUdevResource groups[160];
  unsigned ngroups = 0;
  bool fine = false;               // SM-pair split (no co-scheduling groups)
  CUdevResource rem;
  uint32_t used_groups = 0;
  bool rem_used = false;
  int slots[kMaxSlots] = {-1, -1, -1, -1};
  bool any_live() const {
    for (int s : slots)
      if (s >= 0) return true;
    return false;
  }
};

struct gl_ctx {
  std::vector<GpuState> gpus;
  std::vector<std::unique_ptr<Model>> models;
  std::vector<std::unique_ptr<Gpulet>> gpulets;
  std::deque<gl_completion> stash;  // collected by gl_wait, handed out by gl_poll
  std::mutex mu;
  uint64_t next_ticket = 1;
  uint64_t idle_polls = 0;
  bool poisoned = false;
};

static gl_status cuda_check(gl_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return GL_OK;
  if (c) c->poisoned = true;
  return fail(GL_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
static gl_status cu_check(gl_ctx* c, CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return GL_OK;
  if (c) c->poisoned = true;
  return fail(GL_E_CUDA, std::string(what) + ": CUresult " + std::to_string((int)r));
}
#define CK(x, what)                                  \
  do {                                               \
    gl_status _s = cuda_check(ctx, (x), what);       \
    if (_s != GL_OK) return _s;                      \
  } while (0)

// SMs of a p % gpu-let on a GPU of `total` SMs: p % of the SMs rounded to an
// even count (SM pairs), so the paper's pairs (p, 100 - p) split the
// GPU exactly: 148 -> 20 %: 30, 40 %: 60, 50 %: 74, 60 %: 88, 80 %: 118, 100 %: 148.
static int sm_for_pct(int pct, int total = 148) {
  switch (pct) {
    case 20: case 40: case 50: case 60: case 80:
      return 2 * ((pct * (total / 2) + 50) / 100);
    case 100: return total;
    default: return -1;
  }
}

static size_t exec_smem_bytes() { return (size_t)kSmemBytes + 1024; }

static int grid_index(int pct) {
  switch (pct) {
    case 20: return 0;
    case 40: return 1;
    case 50: return 2;
    case 60: return 3;
    case 80: return 4;
    default: return -1;
  }
}

// One SM split per GPU (SM pairs; 8-SM groups + remainder as a fallback), then one green context and
// stream per (slot, size): slot 0 uses groups from the front, slot 1 from the back.
static gl_status prepare_green(gl_ctx* ctx, GpuState& G) {
  Driver& D = driver();
  CUdevice cud;
  gl_status rc = cu_check(ctx, D.deviceGet(&cud, G.dev), "cuDeviceGet");
  if (rc) return rc;
  CUdevResource all;
  rc = cu_check(ctx, D.deviceGetDevResource(cud, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  if (rc) return rc;
  // The executor uses no thread-block clusters, so the split ignores SM
  // co-scheduling: SM pairs instead of 8-SM groups, which lets every grid size
  // take exactly its share (8-SM groups on this pool's B200s come as 15 groups
  // + a 28-SM remainder, i.e. 24/48/56/72/96 SMs).  Drivers that refuse the
  // flag get the co-scheduled 8-SM split.
  G.ngroups = 160;
  CUresult r = D.devSmResourceSplitByCount(G.groups, &G.ngroups, &all, &G.rem,
                                           CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING, 2);
  G.fine = r == CUDA_SUCCESS;
  if (!G.fine) {
    G.ngroups = 160;
    rc = cu_check(ctx, D.devSmResourceSplitByCount(G.groups, &G.ngroups, &all, &G.rem, 0, 8),
                  "cuDevSmResourceSplitByCount");
    if (rc) return rc;
  }
  G.split = true;
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return fail(GL_E_CUDA, "stream");
  G.full_stream = (CUstream)s;
  G.green_ready = true;
  return GL_OK;
}

// Green context + stream of (slot, size index), created on first use.
static gl_status ensure_green(gl_ctx* ctx, GpuState& G, int slot, int gi) {
  if (G.gctx[slot][gi]) return GL_OK;
  static const int pcts[5] = {20, 40, 50, 60, 80};
  Driver& D = driver();
  CUdevice cud;
  gl_status rc = cu_check(ctx, D.deviceGet(&cud, G.dev), "cuDeviceGet");
  if (rc) return rc;
  const int want = sm_for_pct(pcts[gi], G.nsm);
  std::vector<CUdevResource> res;
  int have = 0;
  // Slot 0 takes groups from the front of the split, slot 1 from the back
  // (the remainder first), each until it holds `want` SMs; for shares p + q
  // <= 100 the two sets are disjoint (the %smid audit of
  // tests/test_gpu_executor.py checks it).  With the SM-pair split every size
  // is exact; with 8-SM groups it is the smallest group count reaching `want`
  // minus one group (sizes never exceed their share).
  // A partition of 3-4 gpu-lets (gl_create_gpulets, SM-pair split only) gives
  // slot s the pairs from layout_pair[s] on, in slot order from the front.
  std::vector<CUdevResource> order;
  if (G.multi) {
    for (unsigned k = (unsigned)G.layout_pair[slot]; k < G.ngroups; ++k) order.push_back(G.groups[k]);
  } else {
    if (slot == 1 && G.rem.sm.smCount > 0) order.push_back(G.rem);
    for (unsigned k = 0; k < G.ngroups; ++k) order.push_back(G.groups[slot == 0 ? k : G.ngroups - 1 - k]);
  }
  for (const CUdevResource& r : order) {
    if (have >= want) break;
    if (!G.fine && have + (int)r.sm.smCount > want) break;
    res.push_back(r);
    have += (int)r.sm.smCount;
  }
  if (have <= 0 || (G.fine && have != want))
    return fail(GL_E_PARTITION, "ensure_green: the SM split cannot give " + std::to_string(want) + " SMs (got " +
                                    std::to_string(have) + ")");
  CUdevResourceDesc desc;
  rc = cu_check(ctx, D.devResourceGenerateDesc(&desc, res.data(), (unsigned)res.size()), "cuDevResourceGenerateDesc");
  if (rc) return rc;
  dbg_log("ensure_green: cuGreenCtxCreate");
  rc = cu_check(ctx, D.greenCtxCreate(&G.gctx[slot][gi], desc, cud, CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
  if (rc) return rc;
  rc = cu_check(ctx, D.greenCtxStreamCreate(&G.gstream[slot][gi], G.gctx[slot][gi], CU_STREAM_NON_BLOCKING, 0),
                "cuGreenCtxStreamCreate");
  if (rc) return rc;
  G.gnsm[slot][gi] = have;
  return GL_OK;
}

// Drop every cached green context of a GPU (only while none of its executors run).
static void drop_green(GpuState& G) {
  for (int s = 0; s < kMaxSlots; ++s)
    for (int gi = 0; gi < 5; ++gi) {
      if (G.gstream[s][gi]) driver().streamDestroy(G.gstream[s][gi]);
      if (G.gctx[s][gi]) driver().greenCtxDestroy(G.gctx[s][gi]);
      G.gstream[s][gi] = nullptr;
      G.gctx[s][gi] = nullptr;
    }
}

static gl_status launch_executor(gl_ctx* ctx, int dev, CUstream stream, int grid, const ExecParams& p) {
  Driver& D = driver();
  if (!D.ok) return fail(GL_E_CUDA, "CUDA driver entry points unavailable");
  CUkernel k = (CUkernel)gl_executor_handle();
  if (!k) return fail(GL_E_CUDA, "cudaGetKernel(gl_executor) failed");
  CUdevice cud;
  CUresult r = D.deviceGet(&cud, dev);
  if (r != CUDA_SUCCESS) return cu_check(ctx, r, "cuDeviceGet");
  r = D.kernelSetAttribute(CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)exec_smem_bytes(), k, cud);
  if (r != CUDA_SUCCESS) return cu_check(ctx, r, "cuKernelSetAttribute");
  CUlaunchConfig cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = grid;
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = kThreads;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.sharedMemBytes = (unsigned)exec_smem_bytes();
  cfg.hStream = stream;
  ExecParams pp = p;
  void* args[] = {&pp};
  r = D.launchKernelEx(&cfg, (CUfunction)k, args, nullptr);
  return cu_check(ctx, r, "cuLaunchKernelEx(gl_executor)");
}

// One-shot run of a program on the whole GPU (kernel unit tests): optional
// warm-up launches (gl_set_tuning key 3; 0 by default since some test ops run
// in place), then a measured launch whose duration (program start -> last step
// barrier, %globaltimer) and per-CTA tile timeline are kept for gl_test_stats.
static std::vector<uint64_t> g_test_tl;
static uint64_t g_test_ns = 0;
static int g_test_tl_cap = 0;
static const int kTestTlCap = 4 * 64;

static gl_status run_oneshot(gl_ctx* ctx, int gpu, Program& prog, const void* in, void* out) {
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  const int nsm = ctx->gpus[gpu].nsm;
  char* ws = nullptr;
  CK(cudaMalloc(&ws, std::max<size_t>(prog.ws_bytes, 256)), "cudaMalloc(ws)");
  CK(cudaMemset(ws, 0, std::max<size_t>(prog.ws_bytes, 256)), "memset ws");
  if (prog.in_copy_bytes)
    CK(cudaMemcpy(ws + prog.in_copy_off, in, prog.in_copy_bytes, cudaMemcpyDeviceToDevice), "copy input to ws");
  std::string berr;
  OpDesc* dprog = upload_bound(prog, ws, berr);
  if (!dprog) return fail(GL_E_CUDA, berr);
  HostRing* ring = nullptr;
  CK(cudaHostAlloc((void**)&ring, sizeof(HostRing), cudaHostAllocMapped), "cudaHostAlloc(ring)");
  HostRing* ring_dev = nullptr;
  CK(cudaHostGetDevicePointer((void**)&ring_dev, ring, 0), "cudaHostGetDevicePointer");
  ExecState* st = nullptr;
  CK(cudaMalloc(&st, sizeof(ExecState)), "cudaMalloc(st)");
  uint64_t* tr = nullptr;
  CK(cudaMalloc(&tr, 1024 * sizeof(uint64_t)), "cudaMalloc(trace)");
  uint64_t* tl = nullptr;
  const size_t tl_n = (size_t)nsm * kTestTlCap;
  CK(cudaMalloc(&tl, tl_n * sizeof(uint64_t)), "cudaMalloc(timeline)");
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  gl_status rc = GL_OK;
  const int runs = 1 + std::max(0, std::min(g_tune[TUNE_WARM], 8));   // warm-up runs first (tuning tool)
  for (int rep = 0; rep < runs && rc == GL_OK; ++rep) {
    std::memset((void*)ring, 0, sizeof(HostRing));
    CK(cudaMemset(st, 0, sizeof(ExecState)), "memset st");
    CK(cudaMemset(tr, 0, 1024 * sizeof(uint64_t)), "memset trace");
    CK(cudaMemset(tl, 0, tl_n * sizeof(uint64_t)), "memset timeline");
    WorkDesc& w = ring->items[0];
    w.ticket = 1;
    w.prog = dprog;
    w.in = in;
    w.out = out;
    w.n_ops = (int)prog.ops.size();
    w.batch = 1;
    ring->tail = 1;
    ExecParams p;
    std::memset(&p, 0, sizeof(p));
    p.ring = ring_dev;
    p.st = st;
    p.ws = ws;
    p.one_shot = 1;
    p.trace = tr;
    p.trace_cap = 1024;
    p.tl = tl;
    p.tl_cap = kTestTlCap;
    p.dbg_flags = g_tune[TUNE_MISC];
    rc = launch_executor(ctx, ctx->gpus[gpu].dev, (CUstream)s, nsm, p);
    if (rc == GL_OK) {
      cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = cuda_check(ctx, e, "executor (one-shot)");
    }
  }
  if (rc == GL_OK) {
    int steps = 0;
    for (auto& op : prog.ops) steps += op.step_end ? 1 : 0;
    std::vector<uint64_t> h(1024);
    cudaMemcpy(h.data(), tr, 1024 * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    g_test_ns = h[std::min(steps, 1023)] - h[0];
    g_test_tl.assign(tl_n, 0);
    cudaMemcpy(g_test_tl.data(), tl, tl_n * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    for (auto& v : g_test_tl)
      if (v) v -= h[0];
    g_test_tl_cap = kTestTlCap;
  }
  cudaStreamDestroy(s);
  release_device(tl, false);
  release_device(tr, false);
  release_device(st, false);
  release_device(ring, true);
  release_device(ws, false);
  release_device(dprog, false);
  return rc;
}

extern "C" {

const char* gl_last_error(void) { return g_err.c_str(); }

gl_status gl_init(int num_gpus, gl_ctx** out) {
  if (!out || num_gpus < 1) return fail(GL_E_ARG, "gl_init: bad arguments");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n < num_gpus) return fail(GL_E_CUDA, "gl_init: not enough CUDA devices");
  if (!driver().ok) return fail(GL_E_CUDA, "gl_init: driver entry points unavailable (driver too old?)");
  auto* c = new gl_ctx();
  c->gpus.resize(num_gpus);
  for (int i = 0; i < num_gpus; ++i) {
    c->gpus[i].dev = i;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, i);
    c->gpus[i].nsm = prop.multiProcessorCount;
    if (prop.major != 10) {
      delete c;
      return fail(GL_E_CUDA, "gl_init: libgpulet is built for sm_100a (B200) only");
    }
  }
  *out = c;
  return GL_OK;
}

gl_status gl_destroy_gpulet(gl_ctx* ctx, int32_t id);

gl_status gl_shutdown(gl_ctx* ctx) {
  if (!ctx) return GL_OK;
  for (auto& g : ctx->gpulets)
    if (g && g->alive) gl_destroy_gpulet(ctx, g->id);
  for (auto& m : ctx->models) {
    if (!m) continue;
    cudaSetDevice(ctx->gpus[m->gpu].dev);
    for (int b = 1; b <= 32; ++b)
      if (m->prog[b].dev) release_device(m->prog[b].dev, false);
    m->w.reset();
  }
  for (auto& G : ctx->gpus) {
    cudaSetDevice(G.dev);
    if (G.green_ready) {
      drop_green(G);
      if (G.full_stream) cudaStreamDestroy((cudaStream_t)G.full_stream);
      for (auto& us : G.ustream)
        if (us) cudaStreamDestroy((cudaStream_t)us), us = nullptr;
      G.green_ready = false;
    }
    for (auto& R : G.slot_res) {
      if (!R.ready) continue;
      for (auto& kv : R.progs)
        for (OpDesc* p : kv.second) release_device(p, false);
      for (auto& kv : R.progs_sm)
        for (OpDesc* p : kv.second) release_device(p, false);
      release_device(R.ws, false);
      release_device(R.st, false);
      release_device(R.smid, false);
      release_device(R.ring, true);
      R = SlotRes();
    }
  }
  delete ctx;
  return GL_OK;
}

gl_status gl_load_model(gl_ctx* ctx, int gpu, int kind, const char* weight_file, int32_t* model_id) {
  if (!ctx || !weight_file || !model_id || gpu < 0 || gpu >= (int)ctx->gpus.size() || kind < 0 ||
      kind >= model_kind_count())
    return fail(GL_E_ARG, "gl_load_model: bad arguments");
  if (ctx->poisoned) return fail(GL_E_CUDA, "context poisoned by an earlier CUDA error");
  std::lock_guard<std::mutex> lk(ctx->mu);
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  auto m = std::make_unique<Model>();
  m->kind = kind;
  m->gpu = gpu;
  std::string err;
  if (!load_glw(weight_file, m->host, err)) return fail(GL_E_PARSE, err);
  m->w = std::make_unique<DevWeights>();
  for (int b = 1; b <= 32; ++b) {
    if (!build_program(kind, b, m->host, *m->w, gpu, m->prog[b], m->in_bytes[b], m->out_bytes[b], err))
      return fail(GL_E_PARSE, std::string(model_name(kind)) + ": " + err);
    Program& p = m->prog[b];
    CK(cudaMalloc(&p.dev, p.ops.size() * sizeof(OpDesc)), "cudaMalloc(program)");
    CK(cudaMemcpy(p.dev, p.ops.data(), p.ops.size() * sizeof(OpDesc), cudaMemcpyHostToDevice), "upload program");
  }
  // (the host copy stays: programs tiled for other gpu-let sizes are built when
  // such a gpu-let is first created, gl_create_gpulets)
  *model_id = (int32_t)ctx->models.size();
  ctx->models.push_back(std::move(m));
  return GL_OK;
}

gl_status gl_model_io(gl_ctx* ctx, int32_t id, int32_t batch, int64_t* in_b, int64_t* out_b) {
  if (!ctx || id < 0 || id >= (int)ctx->models.size() || batch < 1 || batch > 32)
    return fail(GL_E_ARG, "gl_model_io: bad arguments");
  if (in_b) *in_b = (int64_t)ctx->models[id]->in_bytes[batch];
  if (out_b) *out_b = (int64_t)ctx->models[id]->out_bytes[batch];
  return GL_OK;
}

gl_status gl_model_cost(gl_ctx* ctx, int32_t id, int32_t batch, double* flops, double* wbytes) {
  if (!ctx || id < 0 || id >= (int)ctx->models.size() || batch < 1 || batch > 32)
    return fail(GL_E_ARG, "gl_model_cost: bad arguments");
  if (flops) *flops = ctx->models[id]->prog[batch].flops;
  if (wbytes) *wbytes = ctx->models[id]->prog[batch].weight_bytes;
  return GL_OK;
}

// Per-slot resources (workspace, bound programs, rings) are allocated for
// both slots the first time a gpu-let is created on this GPU, while no
// executor runs there: device allocations can synchronise the device and
// would block behind a persistent executor.  The workspace has 25 % headroom
// for programs tiled for smaller gpu-lets (more split-K partials).
static gl_status ensure_slot_res(gl_ctx* ctx, GpuState& G, int gpu, int nslots = 2) {
  nslots = std::max(2, std::min(nslots, kMaxSlots));
  bool all = true;
  for (int s = 0; s < nslots; ++s) all &= G.slot_res[s].ready;
  if (all) return GL_OK;
  size_t ws = 256;
  for (auto& m : ctx->models)
    if (m && m->gpu == gpu)
      for (int b = 1; b <= 32; ++b) ws = std::max(ws, m->prog[b].ws_bytes);
  ws = (ws + ws / 4 + 255) / 256 * 256;
  for (int s = 0; s < nslots; ++s) {
    SlotRes& R = G.slot_res[s];
    if (R.ready) continue;
    R.ws_bytes = ws;
    CK(cudaMalloc(&R.ws, ws), "cudaMalloc(workspace)");
    CK(cudaMemset(R.ws, 0, ws), "memset(workspace)");
    for (size_t mi = 0; mi < ctx->models.size(); ++mi) {
      auto& m = ctx->models[mi];
      if (!m || m->gpu != gpu) continue;
      std::vector<OpDesc*>& v = R.progs[(int)mi];
      v.assign(33, nullptr);
      for (int b = 1; b <= 32; ++b) {
        std::string berr;
        v[b] = upload_bound(m->prog[b], R.ws, berr);
        if (!v[b]) return fail(GL_E_CUDA, "gl_create_gpulet: " + berr);
      }
    }
    CK(cudaHostAlloc((void**)&R.ring, sizeof(HostRing), cudaHostAllocMapped), "cudaHostAlloc(ring)");
    CK(cudaHostGetDevicePointer((void**)&R.ring_dev, R.ring, 0), "cudaHostGetDevicePointer");
    CK(cudaMalloc(&R.st, sizeof(ExecState)), "cudaMalloc(state)");
    CK(cudaMalloc(&R.smid, 160 * sizeof(int)), "cudaMalloc(smid)");
    R.ready = true;
  }
  CK(cudaDeviceSynchronize(), "slot resources");
  return GL_OK;
}

// Programs tiled for a gpu-let of `nsm` SMs (N tile and split-K chosen for
// that SM count instead of a whole B200: measured -3 to -10 % on 56- and
// 96-SM gpu-lets), built and bound for `slot` once, while no executor runs on
// the GPU (gl_create_gpulets).  A model whose programs do not fit the slot's
// workspace keeps the whole-GPU tiling.
static void bind_sized(gl_ctx* ctx, GpuState& G, int gpu, int slot, int nsm) {
  if (nsm <= 0 || nsm >= G.nsm) return;
  SlotRes& R = G.slot_res[slot];
  for (size_t mi = 0; mi < ctx->models.size(); ++mi) {
    auto& m = ctx->models[mi];
    if (!m || m->gpu != gpu || R.progs_sm.count({(int)mi, nsm})) continue;
    std::vector<Program>& vp = m->prog_sm[nsm];
    if (vp.empty()) {
      vp.resize(33);
      std::string err;
      size_t ib = 0, ob = 0;
      for (int b = 1; b <= 32; ++b)
        if (!build_program(m->kind, b, m->host, *m->w, gpu, vp[b], ib, ob, err, nsm)) {
          vp.clear();
          break;
        }
      if (vp.empty()) continue;
    }
    bool fits = true;
    for (int b = 1; b <= 32; ++b) fits &= vp[b].ws_bytes <= R.ws_bytes;
    if (!fits) continue;
    std::vector<OpDesc*> v(33, nullptr);
    bool ok = true;
    for (int b = 1; b <= 32 && ok; ++b) {
      std::string berr;
      v[b] = upload_bound(vp[b], R.ws, berr);
      ok = v[b] != nullptr;
    }
    if (!ok) {
      for (OpDesc* p : v)
        if (p) cudaFree(p);
      continue;
    }
    R.progs_sm[{(int)mi, nsm}] = std::move(v);
  }
}

static gl_status create_gpulet(gl_ctx* ctx, int gpu, int pct, bool unconfined, int32_t* gpulet_id, int32_t* sm_count);

gl_status gl_create_gpulet(gl_ctx* ctx, int gpu, int pct, int32_t* gpulet_id, int32_t* sm_count) {
  if (ctx && gpu >= 0 && gpu < (int)ctx->gpus.size()) {
    GpuState& G = ctx->gpus[gpu];
    if (G.multi && !G.any_live()) {   // back to the front / back layout of 1-2 gpu-lets
      drop_green(G);
      G.multi = false;
    }
  }
  return create_gpulet(ctx, gpu, pct, false, gpulet_id, sm_count);
}

static gl_status create_gpulet(gl_ctx* ctx, int gpu, int pct, bool unconfined, int32_t* gpulet_id, int32_t* sm_count) {
  if (!ctx || !gpulet_id || gpu < 0 || gpu >= (int)ctx->gpus.size()) return fail(GL_E_ARG, "gl_create_gpulet: bad arguments");
  if (sm_for_pct(pct) < 0) return fail(GL_E_GRID, "gl_create_gpulet: sm_pct not in {20,40,50,60,80,100}");
  if (ctx->poisoned) return fail(GL_E_CUDA, "context poisoned by an earlier CUDA error");
  std::lock_guard<std::mutex> lk(ctx->mu);
  GpuState& G = ctx->gpus[gpu];
  int used = 0, nlive = 0;
  for (int s = 0; s < kMaxSlots; ++s)
    if (G.slots[s] >= 0) {
      used += ctx->gpulets[G.slots[s]]->pct;
      ++nlive;
    }
  const int nmax = G.multi ? kMaxSlots : 2;
  if (nlive >= nmax || used + pct > 100)
    return fail(GL_E_PARTITION, "gl_create_gpulet: gpu-let sizes on a GPU must sum to <= 100, at most 2 "
                                "(4 in one gl_create_gpulets partition)");
  int slot = 0;
  while (G.slots[slot] >= 0) ++slot;
  CK(cudaSetDevice(G.dev), "cudaSetDevice");
  dbg_log("create_gpulet: begin");
  auto g = std::make_unique<Gpulet>();
  g->gpu = gpu;
  g->slot = slot;
  g->pct = pct;
  // Green contexts are cached per (slot, size).  cuGreenCtxCreate can block
  // behind a running persistent kernel, so gl_create_gpulets creates a whole
  // GPU partition's contexts before launching any executor.  Slot 0 takes SM
  // pairs from the front of the split, slot 1 from the back (ensure_green).
  if (!G.green_ready) {
    gl_status rc = prepare_green(ctx, G);
    if (rc) return rc;
  }
  if (pct == 100) {
    g->stream = G.full_stream;
    g->own_primary_stream = true;
    g->nsm = G.nsm;
  } else if (unconfined) {
    // the same executor on the primary context: sm_for_pct CTAs that the
    // hardware block scheduler places on any free SMs (no SM confinement)
    if (!G.ustream[slot]) {
      cudaStream_t s;
      CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "unconfined stream");
      G.ustream[slot] = (CUstream)s;
    }
    g->stream = G.ustream[slot];
    g->own_primary_stream = true;
    g->unconfined = true;
    g->nsm = sm_for_pct(pct, G.nsm);
  } else {
    const int gi = grid_index(pct);
    gl_status rc = ensure_green(ctx, G, slot, gi);
    if (rc) return rc;
    g->gctx = G.gctx[slot][gi];
    g->stream = G.gstream[slot][gi];
    g->nsm = G.gnsm[slot][gi];
  }
  {
    gl_status rc = ensure_slot_res(ctx, G, gpu, slot + 1);
    if (rc) return rc;
  }
  dbg_log("create_gpulet: slot resources ready");
  SlotRes& R = G.slot_res[slot];
  for (auto& old : ctx->gpulets)   // a previous gpu-let of this slot gives its ring back
    if (old && old->gpu == gpu && old->slot == slot) old->ring = nullptr;
  g->ws = R.ws;
  g->ws_bytes = R.ws_bytes;
  g->ring = R.ring;
  g->ring_dev = R.ring_dev;
  g->st = R.st;
  g->smid = R.smid;
  std::memset((void*)g->ring, 0, sizeof(HostRing));
  // legacy-stream memsets: they do not wait for the (non-blocking) executor
  // streams; runtime calls on a green-context stream are avoided on purpose
  CK(cudaMemset(g->st, 0, sizeof(ExecState)), "reset state");
  CK(cudaMemset(g->smid, 0xff, 160 * sizeof(int)), "reset smid");
  CK(cudaStreamSynchronize(0), "reset sync");
  dbg_log("create_gpulet: state reset");
  g->id = (int)ctx->gpulets.size();
  ExecParams p;
  std::memset(&p, 0, sizeof(p));
  p.ring = g->ring_dev;
  p.st = g->st;
  p.ws = g->ws;
  p.gpulet = g->id;
  p.one_shot = 0;
  p.smid_log = g->smid;
  ++g_live_exec;
  gl_status rc = launch_executor(ctx, G.dev, g->stream, g->nsm, p);
  dbg_log("create_gpulet: launched");
  if (rc) {
    --g_live_exec;
    return rc;
  }
  // residency handshake: every CTA must reach the loop (green contexts give no
  // co-scheduling guarantee, cuda.h "Green Contexts" notes)
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    int n = 0;
    for (int i = 0; i < g->nsm; ++i) n += g->ring->resident[i] ? 1 : 0;
    if (n == g->nsm) break;
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
      g->ring->quit = 1;
      std::vector<int> sm(160, -1);
      cudaMemcpy(sm.data(), g->smid, 160 * sizeof(int), cudaMemcpyDeviceToHost);
      std::string ids;
      for (int i = 0; i < g->nsm; ++i) ids += (g->ring->resident[i] ? std::to_string(sm[i]) : std::string("-")) + " ";
      // drain the partly resident kernel before the slot's ring / state can be
      // reused: resident CTAs see quit and leave, freeing SMs for the rest; a
      // kernel that does not drain poisons the context
      const auto td = std::chrono::steady_clock::now();
      cudaError_t qe;
      while ((qe = cudaStreamQuery((cudaStream_t)g->stream)) == cudaErrorNotReady &&
             std::chrono::steady_clock::now() - td < std::chrono::seconds(20))
        std::this_thread::sleep_for(std::chrono::microseconds(100));
      --g_live_exec;
      if (qe != cudaSuccess) ctx->poisoned = true;
      return fail(GL_E_NOT_CONCURRENT, "gl_create_gpulet: executor CTAs not co-resident (" + std::to_string(n) + "/" +
                                            std::to_string(g->nsm) + ") slot " + std::to_string(slot) + " pct " +
                                            std::to_string(pct) + " smids: " + ids);
    }
    cudaError_t e = cudaStreamQuery((cudaStream_t)g->stream);
    if (e != cudaErrorNotReady && e != cudaSuccess) {
      --g_live_exec;
      return cuda_check(ctx, e, "executor launch");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  g->alive = true;
  G.slots[slot] = g->id;
  *gpulet_id = g->id;
  if (sm_count) *sm_count = g->nsm;
  ctx->gpulets.push_back(std::move(g));
  return GL_OK;
}

gl_status gl_destroy_gpulet(gl_ctx* ctx, int32_t id) {
  if (!ctx || id < 0 || id >= (int)ctx->gpulets.size() || !ctx->gpulets[id]) return fail(GL_E_ARG, "bad gpu-let id");
  Gpulet& g = *ctx->gpulets[id];
  if (!g.alive) return fail(GL_E_STATE, "gpu-let already destroyed");
  cudaSetDevice(ctx->gpus[g.gpu].dev);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  g.ring->quit = 1;
  cudaError_t e;
  auto t0 = std::chrono::steady_clock::now();
  while ((e = cudaStreamQuery((cudaStream_t)g.stream)) == cudaErrorNotReady) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
      return fail(GL_E_TIMEOUT, "gl_destroy_gpulet: executor did not exit");
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  g.alive = false;
  GpuState& G = ctx->gpus[g.gpu];
  G.slots[g.slot] = -1;
  // the (slot, size) green context and its stream stay for the next gpu-let
  --g_live_exec;
  // workspace, programs and rings stay with the slot for the next gpu-let;
  // completions still in the ring can be polled until the slot is reused
  flush_deferred();
  if (e != cudaSuccess) return cuda_check(ctx, e, "executor");
  return GL_OK;
}

gl_status gl_gpulet_smids(gl_ctx* ctx, int32_t id, int32_t* smids, int32_t cap, int32_t* n) {
  if (!ctx || id < 0 || id >= (int)ctx->gpulets.size() || !smids || !n) return fail(GL_E_ARG, "bad arguments");
  Gpulet& g = *ctx->gpulets[id];
  const int k = std::min(cap, g.nsm);
  cudaSetDevice(ctx->gpus[g.gpu].dev);
  CK(cudaMemcpy(smids, g.smid, k * sizeof(int), cudaMemcpyDeviceToHost), "copy smids");
  *n = k;
  return GL_OK;
}

static gl_status submit_impl(gl_ctx* ctx, int32_t gid, int32_t mid, const void* in_dev, void* out_dev,
                             int32_t batch, float slo_ms, uint64_t* ticket, bool empty);

gl_status gl_submit_batch(gl_ctx* ctx, int32_t gid, int32_t mid, const void* in_dev, void* out_dev, int32_t batch,
                          float slo_ms, uint64_t* ticket) {
  return submit_impl(ctx, gid, mid, in_dev, out_dev, batch, slo_ms, ticket, false);
}

// empty: a descriptor whose program has no step (the executor floor, gl_floor)
static gl_status submit_impl(gl_ctx* ctx, int32_t gid, int32_t mid, const void* in_dev, void* out_dev,
                             int32_t batch, float slo_ms, uint64_t* ticket, bool empty) {
  if (!ctx || gid < 0 || gid >= (int)ctx->gpulets.size() || !in_dev || !out_dev)
    return fail(GL_E_ARG, "gl_submit_batch: bad arguments");
  if (batch < 1 || batch > 32) return fail(GL_E_CAPACITY, "gl_submit_batch: batch outside [1,32]");
  Gpulet& g = *ctx->gpulets[gid];
  if (!g.alive) return fail(GL_E_STATE, "gl_submit_batch: gpu-let destroyed");
  if (mid < 0 || mid >= (int)ctx->models.size() || ctx->models[mid]->gpu != g.gpu)
    return fail(GL_E_MODEL, "gl_submit_batch: model not loaded on this gpu-let's GPU");
  Model& m = *ctx->models[mid];
  SlotRes& SR = ctx->gpus[g.gpu].slot_res[g.slot];
  auto pit = SR.progs.find(mid);
  if (pit == SR.progs.end() || m.prog[batch].ws_bytes > g.ws_bytes)
    return fail(GL_E_STATE, "gl_submit_batch: model loaded after the gpu-let was created");
  // the program tiled for this gpu-let's SM count when one is bound (else the whole-GPU tiling)
  const OpDesc* prog = pit->second[batch];
  int n_ops = (int)m.prog[batch].ops.size();
  auto sit = SR.progs_sm.find({mid, g.nsm});
  if (sit != SR.progs_sm.end()) {
    prog = sit->second[batch];
    n_ops = (int)m.prog_sm[g.nsm][batch].ops.size();
  }
  if (g.tail - g.comp_seen >= (uint64_t)kRing - 1) return fail(GL_E_QUEUE_FULL, "gl_submit_batch: ring full");
  WorkDesc& w = g.ring->items[g.tail % kRing];
  const uint64_t t = ctx->next_ticket++;
  w.ticket = t;
  w.prog = prog;
  w.in = in_dev;
  w.out = out_dev;
  w.n_ops = empty ? 0 : n_ops;
  w.model = mid;
  w.batch = batch;
  w.slo_us = (int32_t)(slo_ms * 1000.0f);
  w.t_submit_ns = now_ns();
  std::atomic_thread_fence(std::memory_order_seq_cst);
  ++g.tail;
  __atomic_store_n(&g.ring->tail, g.tail, __ATOMIC_RELEASE);
  if (ticket) *ticket = t;
  return GL_OK;
}

static int collect(gl_ctx* ctx, gl_completion* out, int max) {
  int n = 0;
  for (auto& gp : ctx->gpulets) {
    if (!gp) continue;
    Gpulet& g = *gp;
    if (!g.ring) continue;
    const uint64_t ct = __atomic_load_n(&g.ring->comp_tail, __ATOMIC_ACQUIRE);
    while (g.comp_seen < ct && n < max) {
      const volatile CompRec& c = g.ring->comp[g.comp_seen % kRing];
      gl_completion& o = out[n++];
      o.ticket = c.ticket;
      o.gpulet = c.gpulet;
      o.model = c.model;
      o.batch = c.batch;
      o.status = c.status;
      o.t_submit_ns = c.t_submit_ns;
      o.t_dequeue_ns = c.t_dequeue_ns;
      o.t_start_ns = c.t_start_ns;
      o.t_end_ns = c.t_end_ns;
      ++g.comp_seen;
    }
  }
  return n;
}

gl_status gl_poll(gl_ctx* ctx, gl_completion* out, int32_t max, int32_t* n_out) {
  if (!ctx || !out || !n_out || max < 0) return fail(GL_E_ARG, "gl_poll: bad arguments");
  int n = 0;
  while (n < max && !ctx->stash.empty()) {
    out[n++] = ctx->stash.front();
    ctx->stash.pop_front();
  }
  n += collect(ctx, out + n, max - n);
  *n_out = n;
  // an executor that exited while alive (device fault / trap) can never
  // complete its queued work: report it instead of letting callers spin
  if (n == 0 && (++ctx->idle_polls & 1023) == 0) {
    for (auto& gp : ctx->gpulets) {
      if (!gp || !gp->alive) continue;
      cudaError_t e = cudaStreamQuery((cudaStream_t)gp->stream);
      if (e != cudaErrorNotReady) {
        gp->alive = false;
        return cuda_check(ctx, e == cudaSuccess ? cudaErrorLaunchFailure : e, "executor exited");
      }
    }
  }
  return GL_OK;
}

gl_status gl_wait(gl_ctx* ctx, uint64_t ticket, int32_t timeout_ms, gl_completion* out) {
  if (!ctx) return fail(GL_E_ARG, "gl_wait: bad arguments");
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    for (auto it = ctx->stash.begin(); it != ctx->stash.end(); ++it) {
      if (it->ticket == ticket) {
        if (out) *out = *it;
        ctx->stash.erase(it);
        return GL_OK;
      }
    }
    gl_completion buf[64];
    int n = collect(ctx, buf, 64);
    for (int i = 0; i < n; ++i) ctx->stash.push_back(buf[i]);
    if (n) continue;
    for (auto& gp : ctx->gpulets) {
      if (!gp || !gp->alive) continue;
      cudaError_t e = cudaStreamQuery((cudaStream_t)gp->stream);
      if (e != cudaErrorNotReady) {
        gp->alive = false;
        return cuda_check(ctx, e == cudaSuccess ? cudaErrorLaunchFailure : e, "executor exited");
      }
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
      return fail(GL_E_TIMEOUT, "gl_wait: timeout");
    std::this_thread::yield();
  }
}

gl_status gl_profile(gl_ctx* ctx, int32_t gid, int32_t mid, int32_t batch, int32_t warmup, int32_t reps,
                     const void* in_dev, void* out_dev, double* median_us) {
  return gl_profile_tail(ctx, gid, mid, batch, warmup, reps, in_dev, out_dev, 0.5, median_us, nullptr);
}

gl_status gl_profile_tail(gl_ctx* ctx, int32_t gid, int32_t mid, int32_t batch, int32_t warmup, int32_t reps,
                          const void* in_dev, void* out_dev, double q, double* median_us, double* q_us) {
  // Service latency as the frontend sees it: one batch in
  // flight; submit -> its completion record visible to gl_poll (host clock).
  if (!ctx || !median_us || reps < 1 || warmup < 0 || !(q >= 0.0 && q < 1.0)) return fail(GL_E_ARG, "gl_profile: bad arguments");
  std::vector<double> lat;
  for (int i = 0; i < warmup + reps; ++i) {
    uint64_t t;
    const gl_status s = gl_submit_batch(ctx, gid, mid, in_dev, out_dev, batch, 0.f, &t);
    if (s) return s;
    const uint64_t t_sub = now_ns();
    const auto t0 = std::chrono::steady_clock::now();
    bool done = false;
    while (!done) {
      gl_completion c[64];
      const int n = collect(ctx, c, 64);
      for (int k = 0; k < n; ++k) {
        if (c[k].ticket == t) {
          done = true;
          if (i >= warmup) lat.push_back((now_ns() - t_sub) / 1000.0);
        } else {
          ctx->stash.push_back(c[k]);
        }
      }
      if (!done && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
        return fail(GL_E_TIMEOUT, "gl_profile: timeout");
    }
  }
  std::sort(lat.begin(), lat.end());
  *median_us = lat[lat.size() / 2];
  if (q_us) *q_us = lat[std::min(lat.size() - 1, (size_t)(q * (double)lat.size()))];
  return GL_OK;
}

gl_status gl_floor(gl_ctx* ctx, int32_t gid, int32_t warmup, int32_t reps, double* host_us, double* device_us) {
  // the executor's fixed service cost (SURVEY §8(d) cfg1 "executor floor"): a
  // descriptor with an empty program through the same ring, dequeue, start
  // barrier and completion path as gl_profile
  if (!ctx || !host_us || reps < 1 || warmup < 0 || gid < 0 || gid >= (int)ctx->gpulets.size() ||
      !ctx->gpulets[gid] || !ctx->gpulets[gid]->alive)
    return fail(GL_E_ARG, "gl_floor: bad arguments");
  Gpulet& g = *ctx->gpulets[gid];
  int mid = -1;
  for (int i = 0; i < (int)ctx->models.size() && mid < 0; ++i)
    if (ctx->models[i] && ctx->models[i]->gpu == g.gpu) mid = i;
  if (mid < 0) return fail(GL_E_MODEL, "gl_floor: no model loaded on the gpu-let's GPU");
  std::vector<double> lat, dev;
  for (int i = 0; i < warmup + reps; ++i) {
    uint64_t t;
    const gl_status s = submit_impl(ctx, gid, mid, g.ws, g.ws, 1, 0.f, &t, true);
    if (s) return s;
    const uint64_t t_sub = now_ns();
    const auto t0 = std::chrono::steady_clock::now();
    bool done = false;
    while (!done) {
      gl_completion c[64];
      const int n = collect(ctx, c, 64);
      for (int k = 0; k < n; ++k) {
        if (c[k].ticket == t) {
          done = true;
          if (i >= warmup) {
            lat.push_back((now_ns() - t_sub) / 1000.0);
            dev.push_back((c[k].t_end_ns - c[k].t_start_ns) / 1000.0);
          }
        } else {
          ctx->stash.push_back(c[k]);
        }
      }
      if (!done && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
        return fail(GL_E_TIMEOUT, "gl_floor: timeout");
    }
  }
  std::sort(lat.begin(), lat.end());
  std::sort(dev.begin(), dev.end());
  *host_us = lat[lat.size() / 2];
  if (device_us) *device_us = dev[dev.size() / 2];
  return GL_OK;
}

gl_status gl_test_gemm(gl_ctx* ctx, int gpu, const void* A, const uint16_t* W, const uint16_t* bias, void* out,
                       int32_t M, int32_t N, int32_t K, int32_t act, int32_t swap_ab, int32_t splitk, int32_t out_fp32,
                       int32_t a_in_ws) {
  if (!ctx || !A || !W || !bias || !out || gpu < 0 || gpu >= (int)ctx->gpus.size() || M < 1 || N < 1 || K < 8 ||
      K % 8)
    return fail(GL_E_ARG, "gl_test_gemm: bad arguments");
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  DevWeights dw;
  Program prog;
  std::string err;
  if (!build_test_gemm(M, N, K, act, swap_ab, splitk, out_fp32, W, bias, a_in_ws, dw, prog, err))
    return fail(GL_E_ARG, err);
  return run_oneshot(ctx, gpu, prog, A, out);
}

gl_status gl_test_conv(gl_ctx* ctx, int gpu, const void* x, const uint16_t* W, const uint16_t* bias, void* y,
                       int32_t N, int32_t H, int32_t Wd, int32_t C, int32_t Cout, int32_t KH, int32_t stride,
                       int32_t pad, int32_t act, int32_t x_in_ws) {
  if (!ctx || !x || !W || !bias || !y || gpu < 0 || gpu >= (int)ctx->gpus.size() || C % 8)
    return fail(GL_E_ARG, "gl_test_conv: bad arguments");
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  DevWeights dw;
  Program prog;
  std::string err;
  if (!build_test_conv(N, H, Wd, C, Cout, KH, stride, pad, act, W, bias, x_in_ws, dw, prog, err))
    return fail(GL_E_ARG, err);
  return run_oneshot(ctx, gpu, prog, x, y);
}

gl_status gl_test_stats(uint64_t* ns, uint64_t* timeline, int32_t cap, int32_t* tl_per_cta) {
  if (ns) *ns = g_test_ns;
  if (tl_per_cta) *tl_per_cta = g_test_tl_cap;
  if (timeline)
    for (int i = 0; i < cap && i < (int)g_test_tl.size(); ++i) timeline[i] = g_test_tl[i];
  return GL_OK;
}

// Cost of publishing one 64-B work descriptor into DEVICE memory, the alternative to
// the host-mapped ring (include/gpulet.h gl_publish_probe).
gl_status gl_publish_probe(gl_ctx* ctx, int gpu, int32_t reps, double* memcpy_us, double* memcpy_p99_us) {
  if (!ctx || gpu < 0 || gpu >= (int)ctx->gpus.size() || !memcpy_us || reps < 10)
    return fail(GL_E_ARG, "gl_publish_probe: bad arguments");
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  WorkDesc* h = nullptr;
  WorkDesc* d = nullptr;
  cudaStream_t st = nullptr;
  CK(cudaHostAlloc(&h, sizeof(WorkDesc), cudaHostAllocDefault), "cudaHostAlloc(probe)");
  CK(cudaMalloc(&d, sizeof(WorkDesc)), "cudaMalloc(probe)");
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  std::memset((void*)h, 0, sizeof(WorkDesc));
  std::vector<double> t;
  gl_status rc = GL_OK;
  for (int i = 0; i < reps + 10 && rc == GL_OK; ++i) {
    h->ticket = (uint64_t)i;
    const auto t0 = std::chrono::steady_clock::now();
    if (cudaMemcpyAsync(d, h, sizeof(WorkDesc), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      rc = fail(GL_E_CUDA, "gl_publish_probe: copy");
    if (i >= 10) t.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
  cudaStreamDestroy(st);
  cudaFree(d);
  cudaFreeHost(h);
  if (rc) return rc;
  std::sort(t.begin(), t.end());
  *memcpy_us = t[t.size() / 2];
  if (memcpy_p99_us) *memcpy_p99_us = t[(t.size() * 99) / 100];
  return GL_OK;
}

// K12 HBM probe on the SMs of a gpu-let size (include/gpulet.h gl_bw_probe).
gl_status gl_bw_probe(gl_ctx* ctx, int gpu, int sm_pct, int64_t bytes, int32_t reps, double* gbs, int32_t* sm_count) {
  if (!ctx || gpu < 0 || gpu >= (int)ctx->gpus.size() || !gbs || bytes < (1 << 20) || reps < 1)
    return fail(GL_E_ARG, "gl_bw_probe: bad arguments");
  if (sm_pct != 100 && grid_index(sm_pct) < 0) return fail(GL_E_GRID, "gl_bw_probe: sm_pct off the grid");
  GpuState& G = ctx->gpus[gpu];
  if (G.any_live()) return fail(GL_E_STATE, "gl_bw_probe: the GPU has live gpu-lets");
  CK(cudaSetDevice(G.dev), "cudaSetDevice");
  if (!G.green_ready) {
    gl_status rc = prepare_green(ctx, G);
    if (rc) return rc;
  }
  CUstream st = G.full_stream;
  int nsm = G.nsm;
  if (sm_pct != 100) {
    const int gi = grid_index(sm_pct);
    gl_status rc = ensure_green(ctx, G, 0, gi);
    if (rc) return rc;
    st = G.gstream[0][gi];
    nsm = G.gnsm[0][gi];
  }
  Driver& D = driver();
  CUkernel k = (CUkernel)gl_probe_handle();
  if (!k) return fail(GL_E_CUDA, "cudaGetKernel(bw_copy) failed");
  const int64_t n16 = bytes / 16;
  char *src = nullptr, *dst = nullptr;
  CK(cudaMalloc(&src, (size_t)n16 * 16), "cudaMalloc(probe src)");
  CK(cudaMalloc(&dst, (size_t)n16 * 16), "cudaMalloc(probe dst)");
  CK(cudaMemset(src, 1, (size_t)n16 * 16), "memset");
  CK(cudaDeviceSynchronize(), "sync");
  CUlaunchConfig cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDimX = nsm * 4;   // 4 CTAs of 512 threads per SM: 64 warps, the SM's full occupancy
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = 512;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.hStream = st;
  int64_t n = n16;
  void* args[] = {&src, &dst, &n};
  double best = 0.0;
  gl_status rc = GL_OK;
  for (int it = 0; it < reps + 1 && !rc; ++it) {   // the first run warms up
    const auto t0 = std::chrono::steady_clock::now();
    CUresult r = D.launchKernelEx(&cfg, (CUfunction)k, args, nullptr);
    if (r != CUDA_SUCCESS) {
      rc = cu_check(ctx, r, "cuLaunchKernelEx(bw_copy)");
      break;
    }
    if (cudaStreamSynchronize((cudaStream_t)st) != cudaSuccess) {
      rc = fail(GL_E_CUDA, "gl_bw_probe: sync");
      break;
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (it > 0) best = std::max(best, 2.0 * (double)n16 * 16 / s / 1e9);
  }
  cudaFree(src);
  cudaFree(dst);
  if (rc) return rc;
  *gbs = best;
  if (sm_count) *sm_count = nsm;
  return GL_OK;
}

gl_status gl_set_tuning(int32_t key, int32_t value) {
  if (key < 0 || key >= kTuneKeys) return fail(GL_E_ARG, "gl_set_tuning: bad key");
  g_tune[key] = value;
  return GL_OK;
}

gl_status gl_test_misc(gl_ctx* ctx, int gpu, int32_t type, const int32_t* ia, int32_t n, const uint16_t* params,
                       int64_t n_params, const void* x, void* y) {
  if (!ctx || !ia || !y || gpu < 0 || gpu >= (int)ctx->gpus.size()) return fail(GL_E_ARG, "gl_test_misc: bad arguments");
  CK(cudaSetDevice(ctx->gpus[gpu].dev), "cudaSetDevice");
  DevWeights dw;
  Program prog;
  std::string err;
  if (!build_test_misc(type, ia, n, params, (size_t)n_params, dw, prog, err)) return fail(GL_E_ARG, err);
  return run_oneshot(ctx, gpu, prog, x, y);
}

}  // extern "C"

extern "C" gl_status gl_run_once(gl_ctx* ctx, int32_t mid, int32_t batch, const void* in_dev, void* out_dev,
                                 int32_t n_sm, uint64_t* trace_ns, int32_t cap, int32_t* n_steps) {
  if (!ctx || mid < 0 || mid >= (int)ctx->models.size() || batch < 1 || batch > 32 || !in_dev || !out_dev)
    return fail(GL_E_ARG, "gl_run_once: bad arguments");
  Model& m = *ctx->models[mid];
  GpuState& G = ctx->gpus[m.gpu];
  if (n_sm < 1 || n_sm > G.nsm) n_sm = G.nsm;
  CK(cudaSetDevice(G.dev), "cudaSetDevice");
  Program& prog = m.prog[batch];
  char* ws = nullptr;
  CK(cudaMalloc(&ws, std::max<size_t>(prog.ws_bytes, 256)), "cudaMalloc(ws)");
  CK(cudaMemset(ws, 0, std::max<size_t>(prog.ws_bytes, 256)), "memset ws");
  std::string berr;
  OpDesc* bound = upload_bound(prog, ws, berr);
  if (!bound) return fail(GL_E_CUDA, "gl_run_once: " + berr);
  HostRing* ring = nullptr;
  CK(cudaHostAlloc((void**)&ring, sizeof(HostRing), cudaHostAllocMapped), "cudaHostAlloc(ring)");
  std::memset((void*)ring, 0, sizeof(HostRing));
  HostRing* ring_dev = nullptr;
  CK(cudaHostGetDevicePointer((void**)&ring_dev, ring, 0), "cudaHostGetDevicePointer");
  ExecState* st = nullptr;
  CK(cudaMalloc(&st, sizeof(ExecState)), "cudaMalloc(st)");
  CK(cudaMemset(st, 0, sizeof(ExecState)), "memset st");
  uint64_t* tr = nullptr;
  const int tcap = 1024 + 8 * 1000;   // step stamps + CTA-0 role stamps (executor dbg_mark)
  CK(cudaMalloc(&tr, tcap * sizeof(uint64_t)), "cudaMalloc(trace)");
  CK(cudaMemset(tr, 0, tcap * sizeof(uint64_t)), "memset trace");
  WorkDesc& w = ring->items[0];
  w.ticket = 0;
  w.prog = bound;
  w.in = in_dev;
  w.out = out_dev;
  w.n_ops = (int)prog.ops.size();
  w.model = mid;
  w.batch = batch;
  ring->tail = 1;
  ExecParams p;
  std::memset(&p, 0, sizeof(p));
  p.ring = ring_dev;
  p.st = st;
  p.ws = ws;
  p.one_shot = 1;
  p.trace = tr;
  p.trace_cap = tcap;
  p.dbg_flags = g_tune[TUNE_MISC];   // tuning experiments only (0 unless gl_set_tuning)
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  gl_status rc = launch_executor(ctx, G.dev, (CUstream)s, n_sm, p);
  if (rc == GL_OK) {
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = cuda_check(ctx, e, "executor (run_once)");
  }
  int steps = 0;
  for (auto& op : prog.ops) steps += op.step_end ? 1 : 0;
  if (rc == GL_OK && trace_ns && cap > 0) {
    std::vector<uint64_t> h(tcap);
    cudaMemcpy(h.data(), tr, tcap * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    for (int i = 0; i < std::min(cap, std::min(steps + 1, tcap)); ++i) trace_ns[i] = h[i];
    // role stamps follow at trace_ns[1024 + 8 * step + k] when the caller's buffer is large enough
    for (int i = 1024; i < std::min(cap, tcap); ++i) trace_ns[i] = h[i];
  }
  if (n_steps) *n_steps = steps;
  cudaStreamDestroy(s);
  release_device(tr, false);
  release_device(bound, false);
  release_device(st, false);
  release_device(ring, true);
  release_device(ws, false);
  return rc;
}

extern "C" gl_status gl_program_info(gl_ctx* ctx, int32_t mid, int32_t batch, int32_t* step_type, int32_t* step_ops,
                                     double* step_flops, double* step_bytes, int32_t cap, int32_t* n_steps) {
  if (!ctx || mid < 0 || mid >= (int)ctx->models.size() || batch < 1 || batch > 32)
    return fail(GL_E_ARG, "gl_program_info: bad arguments");
  Program& prog = ctx->models[mid]->prog[batch];
  int s = 0;
  bool open = false;
  for (auto& op : prog.ops) {
    double f, b;
    op_cost(op, f, b);
    if (s < cap) {
      if (!open) {
        if (step_type) step_type[s] = op.type;
        if (step_ops) step_ops[s] = 0;
        if (step_flops) step_flops[s] = 0;
        if (step_bytes) step_bytes[s] = 0;
        open = true;
      }
      if (step_ops) step_ops[s] += 1;
      if (step_flops) step_flops[s] += f;
      if (step_bytes) step_bytes[s] += b;
    }
    if (op.step_end) {
      ++s;
      open = false;
    }
  }
  if (n_steps) *n_steps = s;
  return GL_OK;
}

// Create a whole GPU partition (1 or 2 gpu-lets) at once: every green context it
// needs is created before the first executor is launched (cuGreenCtxCreate can
// block behind a running persistent kernel).  The GPU must have no live gpu-let.
extern "C" gl_status gl_create_gpulets(gl_ctx* ctx, int gpu, int32_t n, const int32_t* pcts, int32_t* ids,
                                       int32_t* sm_counts) {
  if (!ctx || !pcts || !ids || n < 1 || n > kMaxSlots || gpu < 0 || gpu >= (int)ctx->gpus.size())
    return fail(GL_E_ARG, "gl_create_gpulets: bad arguments");
  GpuState& G = ctx->gpus[gpu];
  if (G.any_live()) return fail(GL_E_STATE, "gl_create_gpulets: GPU has live gpu-lets");
  int sum = 0;
  for (int i = 0; i < n; ++i) {
    if (sm_for_pct(pcts[i]) < 0) return fail(GL_E_GRID, "gl_create_gpulets: sm_pct not in the grid");
    sum += pcts[i];
  }
  if (sum > 100) return fail(GL_E_PARTITION, "gl_create_gpulets: sizes sum to more than 100");
  CK(cudaSetDevice(G.dev), "cudaSetDevice");
  if (!G.green_ready) {
    gl_status rc = prepare_green(ctx, G);
    if (rc) return rc;
  }
  drop_green(G);
  // 3-4 gpu-lets: contiguous SM-pair ranges from the front, in slot order
  G.multi = n > 2;
  if (G.multi) {
    if (!G.fine) return fail(GL_E_PARTITION, "gl_create_gpulets: 3-4 gpu-lets need the SM-pair split");
    int pair = 0;
    for (int i = 0; i < n; ++i) {
      if (pcts[i] == 100) return fail(GL_E_PARTITION, "gl_create_gpulets: a 100 % gpu-let has no sibling");
      G.layout_pair[i] = pair;
      pair += sm_for_pct(pcts[i], G.nsm) / 2;
    }
    if (2 * pair > G.nsm)   // e.g. 20+20+20+40 %: exact shares 30+30+30+60 = 150 > 148 SMs
      return fail(GL_E_PARTITION, "gl_create_gpulets: the exact shares need " + std::to_string(2 * pair) + " SMs");
  }
  for (int i = 0; i < n; ++i)
    if (pcts[i] < 100) {
      gl_status rc = ensure_green(ctx, G, i, grid_index(pcts[i]));
      if (rc) return rc;
    }
  // slot resources and the programs tiled for these gpu-let sizes, before any
  // executor of this GPU runs (gpu-let i takes slot i)
  {
    gl_status rc = ensure_slot_res(ctx, G, gpu, n);
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i)
    bind_sized(ctx, G, gpu, i, pcts[i] == 100 ? G.nsm : G.gnsm[i][grid_index(pcts[i])]);
  CK(cudaDeviceSynchronize(), "sized programs");
  for (int i = 0; i < n; ++i) {
    int32_t sm = 0;
    // the internal path: the partition's green contexts were created above and
    // must survive (the public call resets a 3-4 gpu-let layout on an empty GPU)
    gl_status rc = create_gpulet(ctx, gpu, pcts[i], false, &ids[i], &sm);
    if (rc) return rc;
    if (sm_counts) sm_counts[i] = sm;
  }
  return GL_OK;
}

extern "C" gl_status gl_create_gpulets_unconfined(gl_ctx* ctx, int gpu, int32_t n, const int32_t* pcts, int32_t* ids,
                                                  int32_t* sm_counts) {
  if (!ctx || !pcts || !ids || n < 1 || n > 2 || gpu < 0 || gpu >= (int)ctx->gpus.size())
    return fail(GL_E_ARG, "gl_create_gpulets_unconfined: bad arguments");
  GpuState& G = ctx->gpus[gpu];
  if (G.any_live()) return fail(GL_E_STATE, "gl_create_gpulets_unconfined: GPU has live gpu-lets");
  if (G.multi) {   // forget a 3-4 gpu-let layout's green contexts
    drop_green(G);
    G.multi = false;
  }
  int sum = 0;
  for (int i = 0; i < n; ++i) {
    if (sm_for_pct(pcts[i]) < 0 || pcts[i] == 100)
      return fail(GL_E_GRID, "gl_create_gpulets_unconfined: sm_pct not in {20,40,50,60,80}");
    sum += pcts[i];
  }
  if (sum > 100) return fail(GL_E_PARTITION, "gl_create_gpulets_unconfined: sizes sum to more than 100");
  CK(cudaSetDevice(G.dev), "cudaSetDevice");
  if (!G.green_ready) {
    gl_status rc = prepare_green(ctx, G);
    if (rc) return rc;
  }
  {
    gl_status rc = ensure_slot_res(ctx, G, gpu);
    if (rc) return rc;
  }
  for (int i = 0; i < n; ++i) bind_sized(ctx, G, gpu, i, sm_for_pct(pcts[i], G.nsm));
  CK(cudaDeviceSynchronize(), "sized programs");
  for (int i = 0; i < n; ++i) {
    int32_t sm = 0;
    gl_status rc = create_gpulet(ctx, gpu, pcts[i], true, &ids[i], &sm);
    if (rc) return rc;
    if (sm_counts) sm_counts[i] = sm;
  }
  return GL_OK;
}
