// K0 gpu-let executor and the layer kernels it runs
// (a8-a12): one persistent kernel per gpu-let, 1 CTA per SM of the gpu-let's
// green context, 288 threads:
//   warps 0-3  producers: implicit-im2col gather (cp.async, zero-fill) of the
//              activation operand + TMA of the weight operand into a 4-stage
//              128B-swizzled smem ring (mbarrier full/empty)
//   warp  8    MMA issuer: one elected thread issues tcgen05.mma (bf16 -> fp32
//              accumulators in TMEM, double-buffered 2 x 256 columns)
//   warps 4-7  epilogue: tcgen05.ld TMEM -> registers, +bias (+residual)
//              -> activation -> bf16/fp32 store (or split-K fp32 reduction)
// Non-GEMM ops (depthwise, pools, LeNet, LayerNorm, attention, softmax) use all
// warps on CUDA cores.  A gpu-let-wide barrier separates the steps of a layer
// program.  Work arrives through a host-mapped ring polled by CTA 0.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "program.h"
#include "ptx.cuh"

using namespace gl;

namespace {

constexpr int kLag = 2;  // producer cp.async groups in flight before arriving

struct Ctx {
  const char* in;
  char* out;
  char* ws;
  uint32_t* cnt;   // the program's completion counters (barrier-free GEMM step joins)
};

// Wait until counter *p reaches `need` (acquire, gpu scope).  A join whose
// producer never completes is a bug: trap after 20 s instead of hanging.
__device__ __noinline__ void wait_count(const uint32_t* p, uint32_t need) {
  uint32_t ns = 64;
  uint64_t t0 = 0;
  while (ld_acquire_gpu_u32(p) < need) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    if (t0 == 0) t0 = globaltimer();
    else if (globaltimer() - t0 > 20ull * 1000000000ull) __trap();
  }
}

__device__ __forceinline__ char* res(const BufRef& b, const Ctx& c) {
  switch (b.kind) {
    case BUF_WS: return c.ws + b.off;
    case BUF_IN: return const_cast<char*>(c.in) + b.off;
    case BUF_OUT: return c.out + b.off;
    case BUF_ABS: return reinterpret_cast<char*>(b.off);
    default: return nullptr;
  }
}

struct Smem {
  uint8_t* a[kStages];   // fixed 4-stage layout (scratch for the non-GEMM ops)
  uint8_t* b[kStages];
  uint8_t* ring;         // GEMM ring: stage s at ring + s * stage_bytes (A 16 KB, then B)
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_base;
  uint8_t* scratch;  // non-GEMM ops reuse the stage area
  uint64_t* att;     // attention barriers: [0] Q/K/V landed, [1] S = QK^T done, [2] O = PV done
  int* epi_flag;     // epilogue broadcast word (split-K last arriver)
  volatile uint64_t* wtag;   // global address of the LeNet parameters resident in scratch (0: none)
  uint8_t* estage;   // epilogue staging: 4 warps x 32 rows x kEpiRowBytes (coalesced stores)
  uint64_t* dbg;     // optional per-step role stamps of CTA 0 (one-shot trace mode)
  int step;          // current step index (for dbg)
  uint64_t* tl;      // optional per-tile timeline of step 0 for this CTA (tuning tool)
  int tl_cap;
  int flags;         // ExecParams::dbg_flags
  GemmArgs* opc;     // shared-memory copy of the current GEMM step's op args (first kOpCache ops)
  int* opn;          //   and their unit counts
  float* ebias;      // epilogue: per-warp fp32 bias of the current tile's columns (8 x 256)
};

__device__ __forceinline__ void tl_mark(const Smem& S, int i, int k) {
  if (S.tl && S.step == 0 && 4 * i + k < S.tl_cap) S.tl[4 * i + k] = globaltimer();
}

// CTA 0 role stamps: [0] producer first tile start, [1] producer all issued,
// [2] MMA first stage acquired, [3] MMA last commit, [4] epilogue first tfull,
// [5] epilogue done, [6] CTA at barrier, [7] barrier released.
__device__ __forceinline__ void dbg_mark(const Smem& S, int k) {
  if (S.dbg && blockIdx.x == 0 && S.step < 1000) S.dbg[S.step * 8 + k] = globaltimer();
}

struct Pipe {
  uint32_t stage = 0, nst = kStages;  // smem ring position and depth of the current GEMM step
  uint32_t bits = 0;              // parity of each ring stage's barrier uses (producer / MMA each keep their own)
  uint32_t acc = 0;               // accumulator uses (MMA / epilogue each keep their own)
  uint32_t att_phase = 0;         // attention barrier parity (every thread tracks it)
  int npend = 0;
  uint32_t pend[kLag];
  int fix = 0;                    // a GEMM step ended: apply its tile / k-block counts after the barrier
};

__device__ __forceinline__ uint32_t par(const Pipe& p) { return (p.bits >> p.stage) & 1u; }

__device__ __forceinline__ void advance(Pipe& p) {
  p.bits ^= 1u << p.stage;
  if (++p.stage == p.nst) p.stage = 0;
}

// ------------------------------------------------------------------ gpu-let barrier
// Split-phase gpu-let barrier: arrive (this CTA's step is done: __syncthreads,
// then thread 0's release-add, which orders the CTA's prior writes, made
// visible CTA-wide by the __syncthreads) and wait (thread 0 acquire-polls: tight
// for the first ~1 us, then with a short back-off for idle executors waiting for
// work; then __syncthreads).  Between the two a CTA may do work that does not
// depend on the other CTAs' step (staging the next step's GEMM arguments).
// (Counters spread over 8 lines, CTA b adding to line b % 8 and polling the sum,
// were measured 1 us per barrier slower: profiles/ab_r4j_barrier_spread_lines.log)
__device__ __forceinline__ void gridsync_arrive(ExecState* st) {
  __syncthreads();
  if (threadIdx.x == 0) red_release_gpu_add_u64((unsigned long long*)&st->barrier, 1ull);
}

__device__ void gridsync_wait(ExecState* st, uint64_t& epoch, bool may_idle) {
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)(epoch + 1) * gridDim.x;
    epoch += 1;
    uint32_t spins = 0, ns = 32;
    uint64_t t0 = 0;
    while (ld_acquire_gpu_u64((volatile uint64_t*)&st->barrier) < target) {
      if (++spins < 256) continue;
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
      if (!may_idle) {
        if (t0 == 0) t0 = globaltimer();
        else if (globaltimer() - t0 > 20ull * 1000000000ull) __trap();
      }
    }
  }
  __syncthreads();
  // The next step's TMA (async proxy) reads what other CTAs stored (generic
  // proxy): the thread that issues a step's TMA loads executes
  // fence.proxy.async.global itself before its first load (tma_role_fence),
  // so the other threads do not wait on the proxy fence here.
}

__device__ void gridsync(ExecState* st, uint64_t& epoch, bool may_idle) {
  gridsync_arrive(st);
  gridsync_wait(st, epoch, may_idle);
}

// ------------------------------------------------------------------ epilogue helpers
__device__ __forceinline__ float act_f(float v, int act) {
  switch (act) {
    case ACT_RELU: return fmaxf(v, 0.f);
    case ACT_GELU: return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
    case ACT_TANH: return tanhf(v);
    default: return v;
  }
}

__device__ __forceinline__ int64_t out_index(const Epilogue& e, int r, int c) {
  return (int64_t)(r / e.rows_per_img) * e.img_stride + (int64_t)(r % e.rows_per_img) * e.ldc + e.col_off + c;
}

// Apply bias / residual / activation to an fp32 value of output element (m, n)
// of D[M,N] and store it.  (r, c) = (m, n), or (n, m) for swap-AB.
__device__ __noinline__ void store_one(const Epilogue& e, const Ctx& X, int m, int n, float v) {
  const __nv_bfloat16* bias = (const __nv_bfloat16*)res(e.bias, X);
  if (bias) v += __bfloat162float(bias[e.bias_on_m ? m : n]);
  const int r = e.transpose ? n : m, c = e.transpose ? m : n;
  const int64_t idx = out_index(e, r, c);
  const __nv_bfloat16* rs = (const __nv_bfloat16*)res(e.res, X);
  if (rs) v += __bfloat162float(rs[idx]);
  v = act_f(v, e.act);
  if (e.out_fp32)
    ((float*)res(e.out, X))[idx] = v;
  else
    ((__nv_bfloat16*)res(e.out, X))[idx] = __float2bfloat16_rn(v);
}

template <int ACT>
__device__ __forceinline__ float act_t(float v) {
  if (ACT == ACT_RELU) return fmaxf(v, 0.f);
  if (ACT == ACT_GELU) return 0.5f * v * (1.f + erff(v * 0.70710678118654752f));
  if (ACT == ACT_TANH) return tanhf(v);
  return v;
}

__device__ __forceinline__ void add_bf16x8(float* v, const uint4& u) {
  const __nv_bfloat162* h = (const __nv_bfloat162*)&u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] += f.x;
    v[2 * i + 1] += f.y;
  }
}

// Request the residual chunk [32 rows x 32 columns] at column `col` into the
// staging rows (cp.async, L2 only): lane (sr, seg) copies 16 B of rows
// it * 8 + sr (it = 0..3) at segment seg of the 64-B row chunk.
__device__ __forceinline__ void res_request(uint8_t* stg, const __nv_bfloat16* rsd, int row0, int M, int64_t ldc,
                                            int64_t col, int lane) {
  const int sr = lane >> 2, seg = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + sr;
    const bool ok = row0 + r < M;
    const __nv_bfloat16* src = ok ? rsd + (row0 + r) * ldc + col + seg * 8 : rsd;
    cp_async16(smem_u32(stg + r * kEpiRowBytes + seg * 16), src, ok ? 16u : 0u);
  }
  cp_async_commit();
}

// One 16-column half h of chunk j (see epi_rows): v holds its accumulators
// (TMEM already waited), sb the chunk's fp32 bias (smem), the lane's staging
// row the chunk's residual (RES).  Returns the bf16 results in o.
template <int ACT, bool RES>
__device__ __forceinline__ void epi_half(const uint32_t (&v)[16], uint32_t sb, bool has_bias, const uint4& r0,
                                         const uint4& r1, int h, uint4 (&o)[2]) {
  float x[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) x[c] = __uint_as_float(v[c]);
  if (has_bias) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 b = lds_f4(sb + h * 64 + k * 16);   // broadcast
      x[4 * k] += b.x, x[4 * k + 1] += b.y, x[4 * k + 2] += b.z, x[4 * k + 3] += b.w;
    }
  }
  if (RES) {
    add_bf16x8(x, r0);
    add_bf16x8(x + 8, r1);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    __nv_bfloat162 hh[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      hh[q] = __floats2bfloat162_rn(act_t<ACT>(x[8 * k + 2 * q]), act_t<ACT>(x[8 * k + 2 * q + 1]));
    o[k] = *(const uint4*)hh;
  }
}

// Warp-collective epilogue of the 32 rows [row0, row0 + 32) of one tile, for
// `nfull` full 32-column chunks starting at output column n00 (bf16 row-major
// output): TMEM -> registers, + bias (+ residual) -> ACT -> bf16.  TMEM is read
// in 16-column halves with the next half's load in flight while the current
// one is processed.  Rows are staged in shared memory so that residual loads
// and output stores move 16 B per lane with four lanes per 64-B row segment.
// The caller put the tile's fp32 bias for these columns in sb and, for RES,
// requested chunk 0's residual into the staging rows before the accumulator
// was ready; chunk j + 1's residual is requested after chunk j's stores.
template <int ACT, bool RES>
__device__ __forceinline__ void epi_rows(const Epilogue& e, const GemmArgs& g, const Ctx& X, uint32_t taddr,
                                         int row0, int n00, int nfull, uint8_t* stg, int lane, bool nostore,
                                         const float* sb, bool has_bias, int flags) {
  const __nv_bfloat16* rsd = (const __nv_bfloat16*)res(e.res, X);
  __nv_bfloat16* outp = (__nv_bfloat16*)res(e.out, X);
  const int64_t ldc = e.ldc;
  const int64_t coff = e.col_off;
  const int M = g.M;
  const int sr = lane >> 2, seg = lane & 3;
  const uint32_t srow = smem_u32(stg) + lane * kEpiRowBytes, sstg = smem_u32(stg), sbs = smem_u32(sb);
  uint32_t va[16], vb[16];
  tmem_ld16_issue(taddr, va);
  tmem_wait_ld16(va);
  const bool direct = (flags & 32) != 0;   // tuning: own-row stores (measured slower than staged)
#pragma unroll 1
  for (int j = 0; j < nfull; ++j) {
    const int n0 = n00 + j * 32;
    tmem_ld16_issue(taddr + j * 32 + 16, vb);
    uint4 rr[4];
    if (RES) {
      // this chunk's residual (staged rows) -> registers; the staging rows are
      // then free, so the next chunk's residual is requested right away
      cp_async_wait<0>();
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) rr[k] = lds128(srow + k * 16);
      __syncwarp();
      if (direct && j + 1 < nfull) res_request(stg, rsd, row0, M, ldc, coff + n0 + 32, lane);
    }
    uint4 oa[2], ob[2];
    epi_half<ACT, RES>(va, sbs + j * 128, has_bias, rr[0], rr[1], 0, oa);
    tmem_wait_ld16(vb);
    if (j + 1 < nfull) tmem_ld16_issue(taddr + (j + 1) * 32, va);
    epi_half<ACT, RES>(vb, sbs + j * 128, has_bias, rr[2], rr[3], 1, ob);
    if (direct) {
      // this lane's row: 64 contiguous bytes
      if (row0 + lane < M && !nostore) {
        uint4* dst = (uint4*)(outp + (row0 + lane) * ldc + coff + n0);
        dst[0] = oa[0], dst[1] = oa[1], dst[2] = ob[0], dst[3] = ob[1];
      }
    } else {
      __syncwarp();
      sts128(srow, oa[0]), sts128(srow + 16, oa[1]), sts128(srow + 32, ob[0]), sts128(srow + 48, ob[1]);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int rw = it * 8 + sr;
        if (row0 + rw < M && !nostore)
          *(uint4*)(outp + (row0 + rw) * ldc + coff + n0 + seg * 8) = lds128(sstg + rw * kEpiRowBytes + seg * 16);
      }
      __syncwarp();
      if (RES && j + 1 < nfull) res_request(stg, rsd, row0, M, ldc, coff + n0 + 32, lane);
    }
    if (j + 1 < nfull) tmem_wait_ld16(va);
  }
}

// ------------------------------------------------------------------ operand gather
struct RowCache {
  int pix[8];   // n * H * W, or -1 if the row is out of range
  int h0[8], w0[8];
};

__device__ __forceinline__ void rowcache_init(RowCache& rc, const Gather& g, int row0, int nrows, int t) {
  const int rr = t >> 3;
  const int HoWo = g.Ho * g.Wo;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int lr = rr + 16 * i;
    const int m = row0 + lr;
    if (lr < nrows && m < g.rows) {
      const int n = m / HoWo, rem = m - n * HoWo;
      const int ho = rem / g.Wo, wo = rem - ho * g.Wo;
      rc.pix[i] = n * g.H * g.W;
      rc.h0[i] = ho * g.stride - g.pad;
      rc.w0[i] = wo * g.stride - g.padw;
    } else {
      rc.pix[i] = -1;
      rc.h0[i] = rc.w0[i] = 0;
    }
  }
}

// Gather one 64-wide K block of `nrows` rows into a 128B-swizzled stage.
__device__ __forceinline__ void gather_kblock(const Gather& g, const __nv_bfloat16* x, const RowCache& rc, int nrows,
                                              int kb, int K_real, uint32_t dst, int t) {
  const int c = t & 7, rr = t >> 3;
  const int k0 = kb * 64 + c * 8;
  const bool kvalid = k0 < K_real;
  const int tap = k0 / g.C;
  const int c0 = k0 - tap * g.C;
  const int kh = tap / g.KW, kw = tap - kh * g.KW;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int lr = rr + 16 * i;
    if (lr >= nrows) break;
    const int hi = rc.h0[i] + kh, wi = rc.w0[i] + kw;
    const bool ok = kvalid && rc.pix[i] >= 0 && hi >= 0 && hi < g.H && wi >= 0 && wi < g.W;
    const __nv_bfloat16* src = ok ? x + ((int64_t)(rc.pix[i] + hi * g.W + wi) * g.lda + c0) : x;
    const uint32_t off = lr * 128 + ((c ^ (lr & 7)) << 4);
    cp_async16(dst + off, src, ok ? 16u : 0u);
  }
}

__device__ __forceinline__ void decode_tile(const GemmArgs& g, int lt, int& mb, int& nb, int& kb0, int& kb1) {
  mb = lt % g.n_mblk;
  const int r = lt / g.n_mblk;
  nb = r % g.n_nblk;
  const int s = r / g.n_nblk;
  const int nkb = g.K_pad / 64;
  kb0 = s * g.kb_per_split;
  kb1 = min(nkb, kb0 + g.kb_per_split);
}


// The ops of a GEMM step with their args served from the shared-memory cache
// (read once per step instead of from global memory on every tile).
struct StepOps {
  const OpDesc* ops;
  const GemmArgs* sg;   // shared copies of ops[0 .. min(n, kOpCache))
  const int* su;
  int n;
  __device__ __forceinline__ const GemmArgs& g(int i) const { return i < kOpCache ? sg[i] : ops[i].g; }
  __device__ __forceinline__ int units(int i) const { return i < kOpCache ? su[i] : ops[i].n_units; }
  __device__ __forceinline__ int locate(int t, int& lt) const {
    int i = 0;
    while (i < n - 1 && t >= units(i)) {
      t -= units(i);
      ++i;
    }
    lt = t;
    return i;
  }
};

// Prefetch what the next step reads first, one step ahead.  prefetch_desc:
// its descriptors into L2 (no loads: issued by all threads at step start).
// prefetch_ops: its tensor maps (this SM's descriptor cache) and, with
// GL_WEIGHT_PF, the weights of its GEMM ops (L2; the range is split over the
// gpu-let's CTAs) -- this reads the descriptors, so one warp issues it where it
// would otherwise idle (the MMA warp after its last tile, a single lane of a
// CUDA-core step).
constexpr int kPfOps = 8;
#ifdef GL_WEIGHT_PF
constexpr uint64_t kPfMaxBytes = 8ull << 20;
#endif
__device__ __forceinline__ void prefetch_desc(const OpDesc* nxt, int n) {
  constexpr int kLines = (int)((sizeof(OpDesc) + 127) / 128);
  const int t = threadIdx.x;
  if (t < n * kLines) {
    const char* p = (const char*)(nxt + t / kLines) + (t % kLines) * 128;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
  }
}
__device__ __forceinline__ void prefetch_ops(const OpDesc* nxt, int n, int lane) {
  if (lane >= n) return;
  const OpDesc* op = nxt + lane;
  const int ty = op->type;
  if ((ty == OP_GEMM && op->g.a_tma != SRC_GATHER) || (ty == OP_ATTENTION && op->g.act_tmap))
    tma_prefetch_desc(&op->tmap_a);
  if (ty == OP_GEMM && op->g.b_tma != SRC_GATHER) tma_prefetch_desc(&op->tmap_b);
#ifdef GL_WEIGHT_PF
  // off: measured to raise the co-located LeNet lane's SLO violations (L2/DRAM
  // interference of the bulk prefetch) more than it saves (tools/serve_ab.py)
  const uint64_t a = op->pf_addr, bytes = op->pf_bytes;
  if (a && bytes && bytes <= kPfMaxBytes) {
    const uint64_t chunk = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    if (lo < bytes) {
      const uint32_t sz = (uint32_t)min(chunk, bytes - lo);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a + lo), "r"(sz) : "memory");
    }
  }
#endif
}

// ------------------------------------------------------------------ GEMM step (K1-K4)
// Roles.  Steps whose operands all come by TMA: warp 9 (one thread) produces,
// warp 8 (one thread) issues tcgen05.mma, warps 0-7 run the epilogue (warp w
// owns TMEM lanes 32*(w%4).. and one half of the tile's columns).  Steps with
// a gathered operand: warps 0-3 gather (cp.async) and issue the TMA half,
// warps 4-7 run the epilogue over all columns.  The smem ring depth follows
// the step's widest N tile: 192 KB / (16 KB + BN x 128 B), at most 8 stages.
// One 64-wide K block of the im2col A operand: 64 / cb TMA im2col loads of
// [128 pixels x cb channels], box j at sa + j * 128 * cb * 2.  k = (tap, c) with
// c fastest, so a box never straddles a tap (cb divides C).  Taps past the
// filter (K padding; the weights there are zero) re-read tap (0, 0) so the smem
// operand stays finite.
struct Im2colGeo {   // register copy of the im2col geometry (no global reloads in the k loop)
  int cb, C, KW, ntaps;
};

__device__ __forceinline__ void im2col_kblock(const Im2colGeo& q, const void* tmap, uint64_t* bar, uint32_t sa, int kb,
                                              int icw, int ich, int icn) {
  for (int j = 0; j < 64 / q.cb; ++j) {
    const int k0 = kb * 64 + j * q.cb;
    int tap = k0 / q.C, c0 = k0 - tap * q.C;
    if (tap >= q.ntaps) tap = 0, c0 = 0;
    const int kh = tap / q.KW, kw = tap - kh * q.KW;
    tma_load_im2col_4d(sa + j * 128 * q.cb * 2, tmap, bar, c0, icw, ich, icn, (uint16_t)kw, (uint16_t)kh);
  }
}

__device__ __forceinline__ Im2colGeo im2col_geo(const GemmArgs& g) {
  Im2colGeo q;
  q.cb = g.a_cb ? g.a_cb : 64;
  q.C = g.ga.C;
  q.KW = g.ga.KW;
  q.ntaps = g.ga.KH * g.ga.KW;
  return q;
}

// UMMA smem descriptor of the A operand for the K=16 step k (0..3) of a stage;
// amode = 64 (128-B swizzle), 32, 16 or 8 (im2col channel box).
__device__ __forceinline__ int a_mode(const GemmArgs& g) {
  return (g.a_tma != SRC_IM2COL || g.a_cb == 0 || g.a_cb == 64) ? 64 : g.a_cb;
}
__device__ __forceinline__ uint64_t a_desc(int amode, uint32_t a0, int k) {
  switch (amode) {
    case 64: return umma_sdesc_sw128(a0 + k * 32);
    case 32: return umma_sdesc(a0 + (k >> 1) * 8192 + (k & 1) * 32, 4, 512, 16);   // SW64, 64-B rows
    case 16: return umma_sdesc(a0 + k * 4096, 6, 256, 16);                        // SW32, 32-B rows
    default: return umma_sdesc(a0 + k * 4096, 0, 128, 2048);                     // no swizzle, 16-B rows
  }
}

__device__ __forceinline__ uint32_t stage_bytes_for(int bn) {
  return (uint32_t)kStageBytesA + (uint32_t)((bn * 128 + 1023) & ~1023);
}

// Barrier-free step join: wait until the producer M blocks holding the A rows
// of tile mb are complete (acquire by the issuing lane; then the async proxy --
// the TMA it issues next -- is ordered after the generic stores it observed).
__device__ __forceinline__ void wait_a_rows(const GemmArgs& g, const Ctx& X, int mb) {
  const uint32_t* c = X.cnt + g.dep_a_off;
  const uint32_t need = (uint32_t)g.dep_a_need;
  const int m0 = mb * 128, m1 = min(g.M, m0 + 128) - 1;
  int lo, hi;
  if (g.a_tma == SRC_TMA) {   // [rows, C]: the producer's own rows
    lo = m0 / 128;
    hi = m1 / 128;
  } else {                    // im2col over NHWC [n, H, W, C]: the input rows the window touches
    const Gather& q = g.ga;
    const int HoWo = q.Ho * q.Wo;
    const int n0 = m0 / HoWo, ho0 = (m0 - n0 * HoWo) / q.Wo;
    const int n1 = m1 / HoWo, ho1 = (m1 - n1 * HoWo) / q.Wo;
    const int h_lo = max(0, ho0 * q.stride - q.pad), h_hi = min(q.H - 1, ho1 * q.stride - q.pad + q.KH - 1);
    lo = ((n0 * q.H + h_lo) * q.W) / 128;
    hi = ((n1 * q.H + h_hi) * q.W + q.W - 1) / 128;
  }
  hi = min(hi, g.dep_a_mblk - 1);
  for (int k = lo; k <= hi; ++k) wait_count(c + k, need);
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Epilogue of one warp over the tile columns [c0, c1) (relative to the tile).
// Waits for the accumulator itself (tfull / parity) after issuing the loads
// that do not depend on it (bias, first residual chunk).
__device__ __forceinline__ void epilogue_cols(const GemmArgs& g, const Ctx& X, const Smem& S, uint32_t taddr, int mb,
                                              int nb, int kb0, int q, int c0, int c1, uint8_t* stg, int lane,
                                              uint64_t* tfull, uint32_t parity, float* sb, uint32_t key,
                                              uint32_t& bkey) {
  const Epilogue& e = g.ep;
  if (g.dep_r_off) {   // residual rows written? (lane 0 acquires; the warp barrier orders the others' reads)
    if (lane == 0) wait_count(X.cnt + g.dep_r_off + mb, (uint32_t)g.dep_r_need);
    __syncwarp();
  }
  const int m = mb * 128 + q * 32 + lane;
  const int nend = min(g.N, (nb + 1) * g.BN);
  c1 = min(c1, nend - nb * g.BN);
  const bool fast = !(S.flags & 1) && e.splitk <= 1 && !e.transpose && !e.out_fp32 && e.rows_per_img >= g.M &&
                    (e.ldc % 8) == 0 && (e.col_off % 8) == 0 && c1 > c0;
  const int nfull = fast ? min(8, (c1 - c0) / 32) : 0;
  const __nv_bfloat16* bias = (const __nv_bfloat16*)res(e.bias, X);
  const bool rs = e.res.kind != BUF_NONE && !(S.flags & 128);   // flag 128: tuning, skip the residual (wrong results)
  const int row0 = mb * 128 + q * 32, n00 = nb * g.BN + c0;
  if (nfull > 0) {
    // the tile's bias columns, fp32 in smem; reloaded only when (op, n block) changes
    // (a CTA's tiles of one op mostly share nb: m blocks vary fastest)
    if (bias && bkey != key) {
      for (int i = lane; i < nfull * 32; i += 32) sb[i] = __bfloat162float(bias[n00 + i]);
      __syncwarp();
      bkey = key;
    }
    if (rs) res_request(stg, (const __nv_bfloat16*)res(e.res, X), row0, g.M, e.ldc, (int64_t)e.col_off + n00, lane);
  }
  mbar_wait(tfull, parity);
  tc_fence_after();
  if (c1 <= c0) return;
  int j0 = c0;   // first column (within the tile) not yet stored
  if (S.flags & 1) {
    for (int j = c0; j < c1; j += 32) {
      float v[32];
      tmem_ld32(taddr + j, v);
      if (v[0] == 1234.5f && v[31] == -1.f) store_one(e, X, m, 0, v[1]);
    }
    return;
  }
  if (e.splitk > 1) {
    const int split = kb0 / g.kb_per_split;
    for (int j = c0; j < c1; j += 32) {
      float v[32];
      tmem_ld32(taddr + j, v);
      const int n0 = nb * g.BN + j;
      const int nn = min(32, c1 - j);
      if (m < g.M) {
        if (e.transpose) {
          float* wp = (float*)res(e.ws, X) + (int64_t)split * g.M * g.N + m;
          for (int c = 0; c < nn; ++c) __stcg(wp + (int64_t)(n0 + c) * g.M, v[c]);
        } else {
          float* wp = (float*)res(e.ws, X) + ((int64_t)split * g.M + m) * g.N;
          if (nn == 32 && (g.N & 3) == 0) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              __stcg((float4*)(wp + n0) + c, make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]));
          } else {
            for (int c = 0; c < nn; ++c) __stcg(wp + n0 + c, v[c]);
          }
        }
      }
    }
    return;
  }
  if (nfull > 0) {
    // bf16 row-major output: warp-collective staged epilogue on the full 32-column chunks
    const uint32_t ta = taddr + c0;
    const bool ns = (S.flags & 2) != 0;
    const bool hb = bias != nullptr;
    switch (e.act * 2 + (rs ? 1 : 0)) {
      case 0: epi_rows<ACT_NONE, false>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 1: epi_rows<ACT_NONE, true>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 2: epi_rows<ACT_RELU, false>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 3: epi_rows<ACT_RELU, true>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 4: epi_rows<ACT_GELU, false>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 5: epi_rows<ACT_GELU, true>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      case 6: epi_rows<ACT_TANH, false>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
      default: epi_rows<ACT_TANH, true>(e, g, X, ta, row0, n00, nfull, stg, lane, ns, sb, hb, S.flags); break;
    }
    j0 = c0 + nfull * 32;
  }
  // remaining (partial / fp32 / transposed / strided) columns, element-wise
  for (int j = j0; j < c1; j += 32) {
    const int n0 = nb * g.BN + j;
    float v[32];
    tmem_ld32(taddr + j, v);
    if (m < g.M)
      for (int c = 0; c < 32 && j + c < c1; ++c) store_one(e, X, m, n0 + c, v[c]);
  }
}

// The step's GEMM arguments (first kOpCache ops) and unit counts into shared
// memory, once per step, by the whole CTA.
__device__ __forceinline__ void stage_gemm_args(const OpDesc* ops, int nops, const Smem& S) {
  constexpr int W = (int)sizeof(GemmArgs) / 4;
  const int nc = min(nops, kOpCache);
  for (int i = threadIdx.x; i < nc * W; i += blockDim.x)
    ((uint32_t*)S.opc)[i] = ((const uint32_t*)&ops[i / W].g)[i % W];
  for (int i = threadIdx.x; i < nc; i += blockDim.x) S.opn[i] = ops[i].n_units;
  __syncthreads();
}

// staged: the arguments were staged between the previous step's barrier arrive
// and wait (run_program).
__device__ void gemm_step(const OpDesc* ops, int nops, const Ctx& X, const Smem& Sio, Pipe& Pio, int n_next,
                          bool staged) {
  // register copies: the k loops must not reload ring state through memory
  // after every asm statement (they all clobber "memory")
  const Smem S = Sio;
  Pipe P = Pio;
#ifdef GL_DBG_START
  if (threadIdx.x == 0) dbg_mark(S, 2);   // instrumented build: step entry
#endif
  if (!staged) stage_gemm_args(ops, nops, S);
#ifdef GL_DBG_START
  if (threadIdx.x == 0) dbg_mark(S, 4);   // instrumented build: step args staged
#endif
  const StepOps so{ops, S.opc, S.opn, nops};
  int total = 0, maxbn = 16;
  bool gstep = false;
  for (int i = 0; i < nops; ++i) {
    total += so.units(i);
    maxbn = max(maxbn, so.g(i).BN);
    gstep |= so.g(i).a_tma == SRC_GATHER || so.g(i).b_tma == SRC_GATHER;
  }
  // A stage of a TMA-only step holds kper consecutive K blocks ([A][B] per K block):
  // one ring wait per kper loads for the producer and per 4·kper MMAs for the
  // issuer (a wait on an mbarrier an async unit signals costs ~250-300 cycles;
  // DESIGN §5): the most K blocks (<= kKPair) that leave the ring kKPairMinStages
  // such stages.
  const uint32_t sbytes1 = stage_bytes_for(maxbn);
  int kper = 1;
  if (!gstep)
    while (kper < kKPair && kRingBytes / ((kper + 1) * sbytes1) >= (uint32_t)kKPairMinStages) ++kper;
  const uint32_t sbytes = sbytes1 * (uint32_t)kper;
  P.nst = min((uint32_t)kMaxStages, (uint32_t)kRingBytes / sbytes);
  P.stage = 0;
  const uint32_t ring = smem_u32(S.ring);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The producer / epilogue roles move between warps from step to step, so
  // every thread ends the step with the ring and accumulator state the
  // participating threads reached: this CTA's tile and k-block counts.
  const uint32_t bits0 = P.bits, acc0 = P.acc;

  if (gstep && warp < 4) {
    // ---------------- gather producers (128 threads; thread 0 also issues the TMA half)
    const int t = threadIdx.x;
    if (t == 0) {
      tma_role_fence();
      dbg_mark(S, 0);
    }
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int lt;
      const int oi = so.locate(tile, lt);
      const OpDesc* op = ops + oi;
      const GemmArgs& g = so.g(oi);
      int mb, nb, kb0, kb1;
      decode_tile(g, lt, mb, nb, kb0, kb1);
      const bool gather = g.a_tma == SRC_GATHER || g.b_tma == SRC_GATHER;
      if (!gather && P.npend) {
        // a TMA-only tile follows gathered ones: publish the lagged stages first
        cp_async_wait<0>();
        fence_proxy_async_smem();
        for (int i = 0; i < P.npend; ++i) mbar_arrive(&S.full[P.pend[i]]);
        P.npend = 0;
      }
      const Gather& gg = g.a_tma ? g.gb : g.ga;
      const int grows = g.a_tma ? g.BN : 128;
      const int grow0 = g.a_tma ? nb * g.BN : mb * 128;
      const __nv_bfloat16* gx = (const __nv_bfloat16*)res(gg.x, X);
      RowCache rc;
      if (gather) rowcache_init(rc, gg, grow0, grows, t);
      int icw = 0, ich = 0, icn = 0;
      if (g.a_tma == SRC_IM2COL && t == 0) {
        const int m0 = mb * 128, HoWo = g.ga.Ho * g.ga.Wo;
        icn = m0 / HoWo;
        const int rem = m0 - icn * HoWo, ho = rem / g.ga.Wo, wo = rem - ho * g.ga.Wo;
        ich = ho * g.ga.stride - g.ga.pad;
        icw = wo * g.ga.stride - g.ga.padw;
      }
      const uint32_t tx = (g.a_tma ? 128 * 128 : 0) + (g.b_tma ? g.BN * 128 : 0);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&S.empty[P.stage], par(P) ^ 1);   // empty[stage]
        const uint32_t sa = ring + P.stage * sbytes, sbb = sa + kStageBytesA;
        if (t == 0) {
          mbar_arrive_expect_tx(&S.full[P.stage], tx);
          if (g.a_tma == SRC_TMA) {
            tma_load_2d(sa, &op->tmap_a, &S.full[P.stage], kb * 64, mb * 128);
          } else if (g.a_tma == SRC_IM2COL) {
            im2col_kblock(im2col_geo(g), &op->tmap_a, &S.full[P.stage], sa, kb, icw, ich, icn);
          }
          if (g.b_tma) tma_load_2d(sbb, &op->tmap_b, &S.full[P.stage], kb * 64, nb * g.BN);
        }
        if (!gather) {
          mbar_arrive(&S.full[P.stage]);
          advance(P);
          continue;
        }
        gather_kblock(gg, gx, rc, grows, kb, g.K_real, g.a_tma ? sbb : sa, t);
        cp_async_commit();
        if (P.npend == kLag) {
          cp_async_wait<kLag>();
          fence_proxy_async_smem();
          mbar_arrive(&S.full[P.pend[0]]);
#pragma unroll
          for (int i = 0; i < kLag - 1; ++i) P.pend[i] = P.pend[i + 1];
          --P.npend;
        }
        P.pend[P.npend++] = P.stage;
        advance(P);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int i = 0; i < P.npend; ++i) mbar_arrive(&S.full[P.pend[i]]);
    P.npend = 0;
    if (t == 0) dbg_mark(S, 1);
  } else if (!gstep && warp >= 9) {
    // ---------------- TMA producers (each warp walks the whole loop and every ring
    // position; warp 9 + p issues the K blocks with index p mod kTmaWarps of this
    // CTA's step, one elected lane per warp)
    const int pw = warp - 9;
    int kbi = 0;
#ifdef GL_DBG_START
    if (pw == 0 && lane == 0) dbg_mark(S, 5);          // instrumented build: before the proxy fence
#endif
    tma_role_fence();
    if (pw == 0 && lane == 0) dbg_mark(S, 0);
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int lt;
      const int oi = so.locate(tile, lt);
      const OpDesc* op = ops + oi;
      const GemmArgs& g = so.g(oi);
      int mb, nb, kb0, kb1;
      decode_tile(g, lt, mb, nb, kb0, kb1);
      int icw = 0, ich = 0, icn = 0;
      if (g.a_tma == SRC_IM2COL) {
        const int m0 = mb * 128, HoWo = g.ga.Ho * g.ga.Wo;
        icn = m0 / HoWo;
        const int rem = m0 - icn * HoWo, ho = rem / g.ga.Wo, wo = rem - ho * g.ga.Wo;
        ich = ho * g.ga.stride - g.ga.pad;
        icw = wo * g.ga.stride - g.ga.padw;
      }
      if (g.dep_a_off) {   // barrier-free join: this tile's A rows complete (lane 0 issues the TMA)
        if (lane == 0) wait_a_rows(g, X, mb);
        __syncwarp();
      }
      const uint32_t tx = 128 * 128 + g.BN * 128;
      const bool a2d = g.a_tma == SRC_TMA;
      const Im2colGeo q = im2col_geo(g);
      const int arow = mb * 128, brow = nb * g.BN;
      const void* tA = &op->tmap_a;
      const void* tB = &op->tmap_b;
      const bool skip = (S.flags & 8) != 0;
      for (int kb = kb0; kb < kb1; kb += kper, ++kbi) {
        if (kbi % kTmaWarps == pw) {
          mbar_wait(&S.empty[P.stage], par(P) ^ 1);
          uint64_t* fb = &S.full[P.stage];
          if (elect_one()) {
            if (skip) {
              mbar_arrive_cnt(fb, 129);
            } else {
              const int nk = min(kper, kb1 - kb);
              uint32_t sa = ring + P.stage * sbytes;
              mbar_arrive_expect_tx(fb, tx * (uint32_t)nk);
              for (int j = 0; j < nk; ++j, sa += sbytes1) {
                if (a2d)
                  tma_load_2d(sa, tA, fb, (kb + j) * 64, arow);
                else
                  im2col_kblock(q, tA, fb, sa, kb + j, icw, ich, icn);
                tma_load_2d(sa + kStageBytesA, tB, fb, (kb + j) * 64, brow);
              }
              mbar_arrive_cnt(fb, 128);
            }
          }
          __syncwarp();
        }
        advance(P);
      }
    }
    if (pw == 0 && lane == 0) dbg_mark(S, 1);
  } else if (warp == 8) {
    // ---------------- MMA issuer (whole warp walks the loop; one elected lane issues)
    const uint32_t tbase = *S.tmem_base;
    const uint64_t bhi = umma_sdesc_sw128(0);
    int ntile = 0, nkb_total = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int lt;
      const int oi = so.locate(tile, lt);
      const GemmArgs& g = so.g(oi);
      int mb, nb, kb0, kb1;
      decode_tile(g, lt, mb, nb, kb0, kb1);
      const uint32_t acc = P.acc & 1, use = P.acc >> 1;
      mbar_wait(&S.tempty[acc], (use & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) tl_mark(S, ntile, 0);
      const uint32_t d = tbase + acc * 256;
      const uint32_t idesc = umma_idesc_bf16(128, g.BN);
      // A descriptor = ahi | ((stage A address + ko[k]) >> 4) for the K=16 step k
      const int amode = a_mode(g);
      const uint64_t ahi = a_desc(amode, 0, 0);
      const uint32_t ko1 = amode == 64 ? 32 : amode == 32 ? 32 : 4096;
      const uint32_t ko2 = amode == 64 ? 64 : 8192;
      const uint32_t ko3 = amode == 64 ? 96 : amode == 32 ? 8224 : 12288;
      const bool do_mma = !(S.flags & 4);
#ifndef GL_DBG_START
      if (tile == (int)blockIdx.x && lane == 0) dbg_mark(S, 2);
#endif
      for (int kb = kb0; kb < kb1; kb += kper) {
        mbar_wait(&S.full[P.stage], par(P));
        if (!(S.flags & 16)) tc_fence_after();
        if (elect_one()) {
          if (do_mma) {
            const int nk = min(kper, kb1 - kb);
            uint32_t a0 = ring + P.stage * sbytes;
            for (int j = 0; j < nk; ++j, a0 += sbytes1) {
              const uint32_t b0 = a0 + kStageBytesA;
              umma_bf16(d, ahi | ((a0 & 0x3FFFF) >> 4), bhi | ((b0 & 0x3FFFF) >> 4), idesc, kb + j > kb0 ? 1u : 0u);
              umma_bf16(d, ahi | (((a0 + ko1) & 0x3FFFF) >> 4), bhi | (((b0 + 32) & 0x3FFFF) >> 4), idesc, 1u);
              umma_bf16(d, ahi | (((a0 + ko2) & 0x3FFFF) >> 4), bhi | (((b0 + 64) & 0x3FFFF) >> 4), idesc, 1u);
              umma_bf16(d, ahi | (((a0 + ko3) & 0x3FFFF) >> 4), bhi | (((b0 + 96) & 0x3FFFF) >> 4), idesc, 1u);
            }
          }
          umma_commit(&S.empty[P.stage]);
        }
        __syncwarp();
        advance(P);
      }
      if (elect_one()) umma_commit(&S.tfull[acc]);
      __syncwarp();
      nkb_total += (kb1 - kb0 + kper - 1) / kper;   // ring stages consumed
      if (lane == 0) tl_mark(S, ntile, 1);
      ++ntile;
      ++P.acc;
    }
    if (lane == 0) {
      dbg_mark(S, 3);
      S.opn[kOpCache] = ntile;
      S.opn[kOpCache + 1] = nkb_total;
    }
    prefetch_ops(ops + nops, n_next, lane);
  } else if (warp < 8) {
    // ---------------- epilogue: warps 4-7 (all columns) or 0-7 (column halves)
    const int q = warp & 3, half = warp < 4 ? 1 : 0;
    const uint32_t tbase = *S.tmem_base;
    uint8_t* stg = S.estage + warp * 32 * kEpiRowBytes;
    float* sbias = S.ebias + warp * 256;
    uint32_t bkey = 0xffffffffu;   // (op, n block) whose bias sbias holds
    const uint32_t arrive_n = gstep ? 2u : 1u;
    int ntile = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      int lt;
      const int oi = so.locate(tile, lt);
      const GemmArgs& g = so.g(oi);
      int mb, nb, kb0, kb1;
      decode_tile(g, lt, mb, nb, kb0, kb1);
      const uint32_t acc = P.acc & 1, use = P.acc >> 1;
      const bool lead = q == 0 && half == 0 && lane == 0;
      const uint32_t taddr = tbase + ((uint32_t)(q * 32) << 16) + acc * 256;
      int c0 = 0, c1 = g.BN;
      if (!gstep) {
        const int split = min(g.BN, ((g.BN / 2) + 31) & ~31);
        c0 = half ? split : 0;
        c1 = half ? g.BN : split;
      }
      if (lead) tl_mark(S, ntile, 2);
#ifndef GL_DBG_START
      if (tile == (int)blockIdx.x && lead) dbg_mark(S, 4);
#endif
      epilogue_cols(g, X, S, taddr, mb, nb, kb0, q, c0, c1, stg, lane, &S.tfull[acc], use & 1, sbias,
                    ((uint32_t)oi << 16) | (uint32_t)nb, bkey);
      if (g.pub_off) {   // this warp's stores of the tile are done: one release per warp
        __syncwarp();
        if (lane == 0) red_release_gpu_add_u32(X.cnt + g.pub_off + mb, 1u);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cnt(&S.tempty[acc], arrive_n);
      if (lead) tl_mark(S, ntile, 3);
      ++ntile;
      ++P.acc;
    }
#ifndef GL_DBG_START
    if (q == 0 && half == 0 && lane == 0) dbg_mark(S, 5);
#endif
  }
  // The ring / accumulator state every thread must leave the step with depends
  // on this CTA's tile and k-block counts, which the MMA warp counted as it
  // walked them; gemm_finish() applies them after the gpu-let barrier, whose
  // __syncthreads makes the counts visible (no extra CTA barrier here).
  // Pio is the CTA's one shared copy: the step leaves bits / acc as it found them
  // (bits0 / acc0); thread 0 records the step's ring depth for gemm_finish.
  (void)bits0;
  (void)acc0;
  if (threadIdx.x == 0) {
    Pio.nst = P.nst;
    Pio.fix = 1;
  }
}

__device__ __forceinline__ void gemm_finish(Pipe& P, const Smem& S) {
  const int my_tiles = S.opn[kOpCache], my_kb = S.opn[kOpCache + 1];
  uint32_t flips = 0;
  for (uint32_t st = 0; st < P.nst; ++st) {
    const uint32_t uses = my_kb / P.nst + (st < my_kb % P.nst ? 1u : 0u);
    flips |= (uses & 1u) << st;
  }
  P.bits ^= flips;
  P.stage = 0;
  P.acc += my_tiles;
  P.fix = 0;
}

// ------------------------------------------------------------------ split-K final
// Sums the fp32 partials ws[s][R][Cc] (output order, see the split-K epilogue)
// over s in order, then + bias (+ residual) -> activation -> store.  8 output
// columns per thread (16-B bf16 stores) when the output mapping allows it.
__device__ __noinline__ void splitk_final(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const Epilogue& e = a.ep;
  const float* ws = (const float*)res(e.ws, X);
  const int R = e.transpose ? a.cols : a.rows, Cc = e.transpose ? a.rows : a.cols;
  const int64_t total = (int64_t)R * Cc;
  const __nv_bfloat16* bias = (const __nv_bfloat16*)res(e.bias, X);
  const __nv_bfloat16* rsd = (const __nv_bfloat16*)res(e.res, X);
  const bool bias_on_c = (e.bias_on_m != 0) == (e.transpose != 0);
  const bool vec = (Cc % 8) == 0 && (e.ldc % 8) == 0 && (e.col_off % 8) == 0 && (e.img_stride % 8) == 0 &&
                   !e.out_fp32 && bias_on_c;
  const int tstride = gridDim.x * blockDim.x;
  if (vec) {
    const int64_t nv = total / 8;
    const int cv = Cc / 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += tstride) {
      const int r = (int)(i / cv), c = (int)(i - (int64_t)r * cv) * 8;
      float v[8];
      const float4* p = (const float4*)(ws + (int64_t)r * Cc + c);
      float4 u0 = __ldcg(p), u1 = __ldcg(p + 1);
      v[0] = u0.x, v[1] = u0.y, v[2] = u0.z, v[3] = u0.w, v[4] = u1.x, v[5] = u1.y, v[6] = u1.z, v[7] = u1.w;
      for (int sp = 1; sp < e.splitk; ++sp) {
        p = (const float4*)(ws + (int64_t)sp * total + (int64_t)r * Cc + c);
        u0 = __ldcg(p), u1 = __ldcg(p + 1);
        v[0] += u0.x, v[1] += u0.y, v[2] += u0.z, v[3] += u0.w, v[4] += u1.x, v[5] += u1.y, v[6] += u1.z,
            v[7] += u1.w;
      }
      if (bias) add_bf16x8(v, *(const uint4*)(bias + c));
      const int64_t idx = out_index(e, r, c);
      if (rsd) add_bf16x8(v, *(const uint4*)(rsd + idx));
      __align__(16) __nv_bfloat16 o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = __float2bfloat16_rn(act_f(v[k], e.act));
      *(uint4*)((__nv_bfloat16*)res(e.out, X) + idx) = *(const uint4*)o;
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += tstride) {
    const int r = (int)(i / Cc), c = (int)(i - (int64_t)r * Cc);
    float v = 0.f;
    for (int sp = 0; sp < e.splitk; ++sp) v += __ldcg(ws + (int64_t)sp * total + i);
    // store_one takes GEMM coordinates (m, n)
    if (e.transpose)
      store_one(e, X, c, r, v);
    else
      store_one(e, X, r, c, v);
  }
}

// ------------------------------------------------------------------ depthwise 3x3 (K5)
// Thread item = (image, output row, strip of STRIP output columns, 8-channel
// group); consecutive threads take consecutive channel groups (16-B coalesced).
// All input vectors of an item are loaded (zero outside the image) before any
// arithmetic so the loads overlap; the strip shares its input columns across
// outputs.  32-bit index math (every tensor here is < 2^31 elements).
__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

template <int STRIDE, int STRIP>
__device__ __forceinline__ void dw_item(const MiscArgs& a, const __nv_bfloat16* __restrict__ x, const float* __restrict__ wsm,
                                        __nv_bfloat16* __restrict__ y, int n, int ho, int wo0, int cg) {
  constexpr int NCOL = (STRIP - 1) * STRIDE + 3;
  uint4 xin[3][NCOL];
  const int wi0 = wo0 * STRIDE - a.pad;
#pragma unroll
  for (int kh = 0; kh < 3; ++kh) {
    const int hi = ho * STRIDE - a.pad + kh;
    const bool hok = hi >= 0 && hi < a.H;
    const __nv_bfloat16* row = x + ((n * a.H + (hok ? hi : 0)) * a.W) * a.C + cg * 8;
#pragma unroll
    for (int j = 0; j < NCOL; ++j) {
      const int wi = wi0 + j;
      const bool ok = hok && wi >= 0 && wi < a.W;
      xin[kh][j] = ok ? __ldg((const uint4*)(row + wi * a.C)) : make_uint4(0u, 0u, 0u, 0u);
    }
  }
  float acc[STRIP][8];
  {
    const float4 b0 = *(const float4*)(wsm + 9 * a.C + cg * 8), b1 = *(const float4*)(wsm + 9 * a.C + cg * 8 + 4);
#pragma unroll
    for (int o = 0; o < STRIP; ++o) {
      acc[o][0] = b0.x, acc[o][1] = b0.y, acc[o][2] = b0.z, acc[o][3] = b0.w;
      acc[o][4] = b1.x, acc[o][5] = b1.y, acc[o][6] = b1.z, acc[o][7] = b1.w;
    }
  }
#pragma unroll
  for (int kh = 0; kh < 3; ++kh)
#pragma unroll
    for (int kw = 0; kw < 3; ++kw) {
      const float4 w0 = *(const float4*)(wsm + (kh * 3 + kw) * a.C + cg * 8);
      const float4 w1 = *(const float4*)(wsm + (kh * 3 + kw) * a.C + cg * 8 + 4);
      const float wf[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int o = 0; o < STRIP; ++o) {
        const uint32_t* xx = (const uint32_t*)&xin[kh][o * STRIDE + kw];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[o][2 * c] = fmaf(bf_lo(xx[c]), wf[2 * c], acc[o][2 * c]);
          acc[o][2 * c + 1] = fmaf(bf_hi(xx[c]), wf[2 * c + 1], acc[o][2 * c + 1]);
        }
      }
    }
#pragma unroll
  for (int o = 0; o < STRIP; ++o) {
    if (wo0 + o >= a.Wo) break;
    __align__(16) __nv_bfloat16 ob[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) ob[c] = __float2bfloat16_rn(act_f(acc[o][c], a.act));
    *(uint4*)(y + ((n * a.Ho + ho) * a.Wo + wo0 + o) * a.C + cg * 8) = *(const uint4*)ob;
  }
}

template <int STRIDE, int STRIP>
__device__ __forceinline__ void dw_loop(const MiscArgs& a, const __nv_bfloat16* x, const float* wsm,
                                        __nv_bfloat16* y) {
  const int CG = a.C / 8, WS = (a.Wo + STRIP - 1) / STRIP;
  const int total = a.N * a.Ho * WS * CG;
  const int stride_t = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride_t) {
    const int cg = i % CG;
    int p = i / CG;
    const int ws = p % WS;
    p /= WS;
    const int ho = p % a.Ho, n = p / a.Ho;
    dw_item<STRIDE, STRIP>(a, x, wsm, y, n, ho, ws * STRIP, cg);
  }
}

// Weights ([9][C] tap-major) and bias are expanded to fp32 in shared memory
// once per CTA (the GEMM ring is idle during this step).
__device__ __noinline__ void dwconv(const OpDesc* op, const Ctx& X, uint8_t* scratch) {
  const MiscArgs& a = op->m;
  const __nv_bfloat16* x = (const __nv_bfloat16*)res(a.x, X);
  const __nv_bfloat16* w = (const __nv_bfloat16*)res(a.w, X);
  const __nv_bfloat16* b = (const __nv_bfloat16*)res(a.b, X);
  __nv_bfloat16* y = (__nv_bfloat16*)res(a.y, X);
  float* wsm = (float*)scratch;   // [9][C] weights then [C] bias
  for (int i = threadIdx.x; i < 10 * a.C; i += blockDim.x)
    wsm[i] = __bfloat162float(i < 9 * a.C ? w[i] : b[i - 9 * a.C]);
  __syncthreads();
  if (a.stride == 1)
    dw_loop<1, 2>(a, x, wsm, y);
  else
    dw_loop<2, 2>(a, x, wsm, y);
  __syncthreads();
}

// ------------------------------------------------------------------ max pool (K6)
// One output pixel x 8 channels per thread item; the K x K window's vectors are
// all loaded (predicated) before the max so the loads overlap.  Max commutes
// with bf16 rounding, so bf16 max is exact.
template <int K>
__device__ __forceinline__ void maxpool_k(const MiscArgs& a, const __nv_bfloat16* __restrict__ x,
                                          __nv_bfloat16* __restrict__ y) {
  const int CG = a.C / 8;
  const int total = a.N * a.Ho * a.Wo * CG;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cg = i % CG;
    int p = i / CG;
    const int wo = p % a.Wo;
    p /= a.Wo;
    const int ho = p % a.Ho, n = p / a.Ho;
    const int h0 = ho * a.stride - a.pad, w0 = wo * a.stride - a.pad;
    uint4 v[K * K];
    bool ok[K * K];
#pragma unroll
    for (int kh = 0; kh < K; ++kh)
#pragma unroll
      for (int kw = 0; kw < K; ++kw) {
        const int hi = h0 + kh, wi = w0 + kw;
        ok[kh * K + kw] = hi >= 0 && hi < a.H && wi >= 0 && wi < a.W;
        v[kh * K + kw] = ok[kh * K + kw] ? __ldg((const uint4*)(x + ((n * a.H + hi) * a.W + wi) * a.C + cg * 8))
                                         : make_uint4(0u, 0u, 0u, 0u);
      }
    __nv_bfloat162 mx[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) mx[c] = __floats2bfloat162_rn(-INFINITY, -INFINITY);
#pragma unroll
    for (int t = 0; t < K * K; ++t) {
      if (!ok[t]) continue;
      const __nv_bfloat162* xx = (const __nv_bfloat162*)&v[t];
#pragma unroll
      for (int c = 0; c < 4; ++c) mx[c] = __hmax2(mx[c], xx[c]);
    }
    *(uint4*)(y + ((n * a.Ho + ho) * a.Wo + wo) * a.C + cg * 8) = *(const uint4*)mx;
  }
}

__device__ __noinline__ void maxpool(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const __nv_bfloat16* x = (const __nv_bfloat16*)res(a.x, X);
  __nv_bfloat16* y = (__nv_bfloat16*)res(a.y, X);
  if (a.k == 2)
    maxpool_k<2>(a, x, y);
  else if (a.k == 3)
    maxpool_k<3>(a, x, y);
  else
    __trap();
}

// ------------------------------------------------------------------ global avg pool (K6)
__device__ __noinline__ void avgpool(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const __nv_bfloat16* x = (const __nv_bfloat16*)res(a.x, X);
  __nv_bfloat16* y = (__nv_bfloat16*)res(a.y, X);
  const int CG = a.C / 8, HW = a.H * a.W;
  const int total = a.N * CG;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int cg = i % CG, n = i / CG;
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < HW; ++p) {
      const uint4 xv = *(const uint4*)(x + ((int64_t)n * HW + p) * a.C + cg * 8);
      const __nv_bfloat16* xx = (const __nv_bfloat16*)&xv;
#pragma unroll
      for (int c = 0; c < 8; ++c) s[c] += __bfloat162float(xx[c]);
    }
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) o[c] = __float2bfloat16_rn(s[c] / (float)HW);
    *(uint4*)(y + (int64_t)n * a.C + cg * 8) = *(const uint4*)o;
  }
}

// ------------------------------------------------------------------ LeNet-5 fused (K7)
__device__ __forceinline__ float bfr(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

template <int K, int J>
__device__ __forceinline__ void lenet_fc4(const float* in, const __nv_bfloat16* w, const __nv_bfloat16* bias, float* out,
                                          int warp, int nw, int lane) {
  static_assert(J % 4 == 0, "groups of 4 neurons");
  for (int j0 = warp * 4; j0 < J; j0 += nw * 4) {
    float s[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = lane; k < K; k += 32) {
      const float v = in[k];
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] = fmaf(v, __bfloat162float(w[(j0 + q) * K + k]), s[q]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
    const float r = lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3];
    if (lane < 4) out[j0 + lane] = bfr(fmaxf(r + __bfloat162float(bias[j0 + lane]), 0.f));
  }
}

__device__ __noinline__ void lenet(const OpDesc* op, const Ctx& X, uint8_t* scratch, volatile uint64_t* wtag) {
  // One CTA per image (grid-stride); the packed bf16 parameters (123 KB) are
  // staged in shared memory once per CTA, activations stay in shared memory
  // in fp32 (rounded to bf16 where the oracle rounds: after each ReLU, C1.4).
  const MiscArgs& a = op->m;
  if ((int)blockIdx.x >= a.N) return;
  const __nv_bfloat16* x = (const __nv_bfloat16*)res(a.x, X);
  const __nv_bfloat16* Wg = (const __nv_bfloat16*)res(a.w, X);  // packed params in manifest order
  float* y = (float*)res(a.y, X);
  constexpr int kParams = 61706, kParamVec = (kParams + 7) / 8;
  __nv_bfloat16* W = (__nv_bfloat16*)scratch;
  // The parameters stay resident in shared memory across batches while only
  // LeNet runs on this gpu-let (wtag = the global address they were staged
  // from; any other op clears it, run_program): a steady LeNet lane reads
  // 123 KB per CTA once instead of once per batch.
  const __nv_bfloat16 *w1 = W, *b1 = w1 + 150, *w2 = b1 + 6, *b2 = w2 + 2400, *f1 = b2 + 16, *fb1 = f1 + 48000,
                      *f2 = fb1 + 120, *fb2 = f2 + 10080, *f3 = fb2 + 84, *fb3 = f3 + 840;
  float* img = (float*)(scratch + kParamVec * 16);   // 28*28
  float* c1 = img + 784;          // 28*28*6 pre-pool (relu, bf16-rounded)
  float* p1 = c1 + 4704;          // 14*14*6
  float* c2 = p1 + 1176;          // 10*10*16 pre-pool
  float* p2 = c2 + 1600;          // 5*5*16 (NHWC flatten)
  float* h1 = p2 + 400;           // 120
  float* h2 = h1 + 120;           // 84
  // conv weights tap-major in fp32 (staged with the parameters): a thread
  // computing all output channels of one pixel reads them as float4 broadcasts
  float* w1t = h2 + 88;           // [25 taps][8] (co 0..5, 2 pad)
  float* w2t = w1t + 25 * 8;      // [150 (tap, ci)][16 co]
  if (*wtag != (uint64_t)(uintptr_t)Wg) {
    for (int i = threadIdx.x; i < kParamVec; i += blockDim.x) ((uint4*)W)[i] = __ldg((const uint4*)Wg + i);
    __syncthreads();
    for (int i = threadIdx.x; i < 25 * 8; i += blockDim.x) {
      const int t = i / 8, co = i % 8;
      w1t[i] = co < 6 ? __bfloat162float(w1[co * 25 + t]) : 0.f;
    }
    for (int i = threadIdx.x; i < 150 * 16; i += blockDim.x) {
      const int k = i / 16, co = i % 16;
      w2t[i] = __bfloat162float(w2[co * 150 + k]);
    }
    __syncthreads();
    if (threadIdx.x == 0) *wtag = (uint64_t)(uintptr_t)Wg;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int n = blockIdx.x; n < a.N; n += gridDim.x) {
    // the image as 98 16-B loads (one round trip when it is read over PCIe
    // from a pinned host ring, gl_serve's zero-copy path)
    if (threadIdx.x < 98) {
      const uint4 u = ((const uint4*)(x + (int64_t)n * 784))[threadIdx.x];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        img[threadIdx.x * 8 + 2 * k] = bf_lo(w4[k]);
        img[threadIdx.x * 8 + 2 * k + 1] = bf_hi(w4[k]);
      }
    }
    __syncthreads();
    for (int px = threadIdx.x; px < 784; px += blockDim.x) {   // conv1 5x5 pad 2 + relu + bf16: one pixel, 6 co
      const int ox = px % 28, oy = px / 28;
      float acc[6];
#pragma unroll
      for (int co = 0; co < 6; ++co) acc[co] = __bfloat162float(b1[co]);
#pragma unroll
      for (int kh = 0; kh < 5; ++kh) {
        const int iy = oy + kh - 2;
        if (iy < 0 || iy >= 28) continue;
#pragma unroll
        for (int kw = 0; kw < 5; ++kw) {
          const int ix = ox + kw - 2;
          if (ix < 0 || ix >= 28) continue;
          const float v = img[iy * 28 + ix];
          const float4 wa = *(const float4*)(w1t + (kh * 5 + kw) * 8);
          const float2 wb = *(const float2*)(w1t + (kh * 5 + kw) * 8 + 4);
          acc[0] = fmaf(v, wa.x, acc[0]), acc[1] = fmaf(v, wa.y, acc[1]), acc[2] = fmaf(v, wa.z, acc[2]);
          acc[3] = fmaf(v, wa.w, acc[3]), acc[4] = fmaf(v, wb.x, acc[4]), acc[5] = fmaf(v, wb.y, acc[5]);
        }
      }
#pragma unroll
      for (int co = 0; co < 6; ++co) c1[px * 6 + co] = bfr(fmaxf(acc[co], 0.f));   // index (oy*28 + ox)*6 + co
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 1176; i += blockDim.x) {   // maxpool 2x2
      const int co = i % 6, px = (i / 6) % 14, py = i / 84;
      const float* q = c1 + ((2 * py) * 28 + 2 * px) * 6 + co;
      p1[i] = fmaxf(fmaxf(q[0], q[6]), fmaxf(q[168], q[174]));
    }
    __syncthreads();
    for (int it = threadIdx.x; it < 200; it += blockDim.x) {   // conv2 5x5 (6->16) + relu + bf16: one pixel, 8 co
      const int hc = it & 1, px = it >> 1;
      const int ox = px % 10, oy = px / 10;
      float acc[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] = __bfloat162float(b2[hc * 8 + k]);
#pragma unroll 5
      for (int kh = 0; kh < 5; ++kh)
#pragma unroll
        for (int kw = 0; kw < 5; ++kw) {
          const float* pp = p1 + ((oy + kh) * 14 + ox + kw) * 6;
          const float* wt = w2t + (kh * 5 + kw) * 6 * 16 + hc * 8;
#pragma unroll
          for (int ci = 0; ci < 6; ++ci) {
            const float v = pp[ci];
            const float4 wa = *(const float4*)(wt + ci * 16), wb = *(const float4*)(wt + ci * 16 + 4);
            acc[0] = fmaf(v, wa.x, acc[0]), acc[1] = fmaf(v, wa.y, acc[1]), acc[2] = fmaf(v, wa.z, acc[2]);
            acc[3] = fmaf(v, wa.w, acc[3]), acc[4] = fmaf(v, wb.x, acc[4]), acc[5] = fmaf(v, wb.y, acc[5]);
            acc[6] = fmaf(v, wb.z, acc[6]), acc[7] = fmaf(v, wb.w, acc[7]);
          }
        }
#pragma unroll
      for (int k = 0; k < 8; ++k) c2[px * 16 + hc * 8 + k] = bfr(fmaxf(acc[k], 0.f));   // index (oy*10 + ox)*16 + co
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 400; i += blockDim.x) {    // maxpool 2x2 -> NHWC flatten (h, w, c)
      const int co = i % 16, px = (i / 16) % 5, py = i / 80;
      const float* q = c2 + ((2 * py) * 10 + 2 * px) * 16 + co;
      p2[i] = fmaxf(fmaxf(q[0], q[16]), fmaxf(q[160], q[176]));
    }
    __syncthreads();
    // fully connected layers: one warp per group of 4 output neurons (4
    // independent accumulation chains), lanes stride over k, shuffle reduction
    lenet_fc4<400, 120>(p2, f1, fb1, h1, warp, nw, lane);
    __syncthreads();
    lenet_fc4<120, 84>(h1, f2, fb2, h2, warp, nw, lane);
    __syncthreads();
    for (int j = warp; j < 10; j += nw) {
      float s = 0.f;
      for (int k = lane; k < 84; k += 32) s = fmaf(h2[k], __bfloat162float(f3[j * 84 + k]), s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) y[(int64_t)n * 10 + j] = s + __bfloat162float(fb3[j]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ LayerNorm rows (K8, K10)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per 768-wide row; 24 values per lane (3 x 16-byte vectors).
__device__ __forceinline__ void ln_row_store(float* v, const __nv_bfloat16* g, const __nv_bfloat16* b, float eps,
                                             __nv_bfloat16* y, int lane) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 24; ++i) s += v[i];
  const float mean = warp_sum(s) * (1.f / 768.f);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    const float d = v[i] - mean;
    q += d * d;
  }
  const float rstd = rsqrtf(warp_sum(q) * (1.f / 768.f) + eps);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int c0 = j * 256 + lane * 8;
    const uint4 gv = *(const uint4*)(g + c0), bv = *(const uint4*)(b + c0);
    const __nv_bfloat16 *gg = (const __nv_bfloat16*)&gv, *bb = (const __nv_bfloat16*)&bv;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      o[c] = __float2bfloat16_rn((v[j * 8 + c] - mean) * rstd * __bfloat162float(gg[c]) + __bfloat162float(bb[c]));
    *(uint4*)(y + c0) = *(const uint4*)o;
  }
}

__device__ __noinline__ void layernorm(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const __nv_bfloat16* x = (const __nv_bfloat16*)res(a.x, X);
  __nv_bfloat16* y = (__nv_bfloat16*)res(a.y, X);
  const __nv_bfloat16 *g = (const __nv_bfloat16*)res(a.g, X), *b = (const __nv_bfloat16*)res(a.b, X);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int nw = gridDim.x * wpb;
  // two rows per warp iteration, both rows' loads issued before either reduction
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < a.rows; r += 2 * nw) {
    const int r2 = r + nw;
    uint4 u[2][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      u[0][j] = __ldcs((const uint4*)(x + (int64_t)r * 768 + j * 256 + lane * 8));
      u[1][j] = r2 < a.rows ? __ldcs((const uint4*)(x + (int64_t)r2 * 768 + j * 256 + lane * 8))
                            : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && r2 >= a.rows) break;
      float v[24];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const __nv_bfloat16* xx = (const __nv_bfloat16*)&u[h][j];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[j * 8 + c] = __bfloat162float(xx[c]);
      }
      ln_row_store(v, g, b, a.eps, y + (int64_t)(h ? r2 : r) * 768, lane);
    }
  }
}

__device__ __noinline__ void embed_ln(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const int32_t* ids = (const int32_t*)res(a.x, X);
  const __nv_bfloat16* word = (const __nv_bfloat16*)res(a.w, X);   // [vocab, 768]
  const __nv_bfloat16* pos = (const __nv_bfloat16*)res(a.aux, X);  // [512, 768] followed by type [2, 768]
  const __nv_bfloat16* typ = pos + 512 * 768;
  __nv_bfloat16* y = (__nv_bfloat16*)res(a.y, X);
  const __nv_bfloat16 *g = (const __nv_bfloat16*)res(a.g, X), *b = (const __nv_bfloat16*)res(a.b, X);
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int r = blockIdx.x * wpb + (threadIdx.x >> 5); r < a.rows; r += gridDim.x * wpb) {
    const int id = ids[r], s = r % a.seq;
    float v[24];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c0 = j * 256 + lane * 8;
      const uint4 wv = *(const uint4*)(word + (int64_t)id * 768 + c0);
      const uint4 pv = *(const uint4*)(pos + (int64_t)s * 768 + c0);
      const uint4 tv = *(const uint4*)(typ + c0);
      const __nv_bfloat16 *ww = (const __nv_bfloat16*)&wv, *pp = (const __nv_bfloat16*)&pv,
                          *tt = (const __nv_bfloat16*)&tv;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        v[j * 8 + c] = __bfloat162float(ww[c]) + __bfloat162float(pp[c]) + __bfloat162float(tt[c]);
    }
    ln_row_store(v, g, b, a.eps, y + (int64_t)r * 768, lane);
  }
}

// ------------------------------------------------------------------ attention (K9)
// Unit = (sequence, head): S = Q K^T / 8 (fp32), softmax fp32, P -> bf16,
// O = P V (fp32) -> bf16.  qkv [b*seq, 3*768]; ctx [b*seq, 768].
__device__ __noinline__ void attention(const OpDesc* op, const Ctx& X, uint8_t* scratch) {
  const MiscArgs& a = op->m;
  const __nv_bfloat16* qkv = (const __nv_bfloat16*)res(a.x, X);
  __nv_bfloat16* ctx = (__nv_bfloat16*)res(a.y, X);
  const int S = a.seq, DH = a.dh, H = a.heads, HD = H * DH;   // 128, 64, 12, 768
  float* Ks = (float*)scratch;                 // [S][DH+1]
  float* Vs = Ks + S * (DH + 1);               // [S][DH]
  __nv_bfloat16* Ps = (__nv_bfloat16*)(Vs + S * DH);  // [S][S+8]
  const int units = a.N * H;
  const int t = threadIdx.x;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int seqi = u / H, h = u % H;
    const __nv_bfloat16* base = qkv + (int64_t)seqi * S * 3 * HD;
    for (int i = t; i < S * DH / 8; i += blockDim.x) {
      const int r = i / (DH / 8), c8 = (i % (DH / 8)) * 8;
      const uint4 kv = *(const uint4*)(base + (int64_t)r * 3 * HD + HD + h * DH + c8);
      const uint4 vv = *(const uint4*)(base + (int64_t)r * 3 * HD + 2 * HD + h * DH + c8);
      const __nv_bfloat16 *kk = (const __nv_bfloat16*)&kv, *vvv = (const __nv_bfloat16*)&vv;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        Ks[r * (DH + 1) + c8 + c] = __bfloat162float(kk[c]);
        Vs[r * DH + c8 + c] = __bfloat162float(vvv[c]);
      }
    }
    __syncthreads();
    if (t < 2 * S) {
      const int i = t >> 1, half = t & 1;
      float q[64];
      const __nv_bfloat16* qp = base + (int64_t)i * 3 * HD + h * DH;
#pragma unroll
      for (int d8 = 0; d8 < 64; d8 += 8) {
        const uint4 qv = *(const uint4*)(qp + d8);
        const __nv_bfloat16* qq = (const __nv_bfloat16*)&qv;
#pragma unroll
        for (int c = 0; c < 8; ++c) q[d8 + c] = __bfloat162float(qq[c]);
      }
      float s[64];
      float mx = -INFINITY;
#pragma unroll 4
      for (int jj = 0; jj < 64; ++jj) {
        const float* kr = Ks + (half * 64 + jj) * (DH + 1);
        float acc = 0.f;
#pragma unroll
        for (int d = 0; d < 64; ++d) acc = fmaf(q[d], kr[d], acc);
        s[jj] = acc * 0.125f;
        mx = fmaxf(mx, s[jj]);
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      float sum = 0.f;
#pragma unroll
      for (int jj = 0; jj < 64; ++jj) {
        s[jj] = expf(s[jj] - mx);
        sum += s[jj];
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      const float inv = 1.f / sum;
#pragma unroll
      for (int jj = 0; jj < 64; ++jj) Ps[i * (S + 8) + half * 64 + jj] = __float2bfloat16_rn(s[jj] * inv);
    }
    __syncthreads();
    if (t < 2 * S) {
      const int i = t >> 1, half = t & 1;
      float o[32];
#pragma unroll
      for (int d = 0; d < 32; ++d) o[d] = 0.f;
      for (int j = 0; j < S; ++j) {
        const float p = __bfloat162float(Ps[i * (S + 8) + j]);
        const float* vr = Vs + j * DH + half * 32;
#pragma unroll
        for (int d = 0; d < 32; ++d) o[d] = fmaf(p, vr[d], o[d]);
      }
      __align__(16) __nv_bfloat16 ob[32];
#pragma unroll
      for (int d = 0; d < 32; ++d) ob[d] = __float2bfloat16_rn(o[d]);
      uint4* dst = (uint4*)(ctx + ((int64_t)seqi * S + i) * HD + h * DH + half * 32);
#pragma unroll
      for (int c = 0; c < 4; ++c) dst[c] = ((const uint4*)ob)[c];
    }
    __syncthreads();
  }
}

// Tensor-core attention (K9): one (sequence, head) unit per CTA iteration.
// TMA brings Q, K, V [128 x 64] (128B-swizzled) from the bound qkv tensor map;
// S = Q K^T is one 128x128x64 UMMA into TMEM columns [0,128); the epilogue warps
// (one query row per thread) read S three times (max, sum, normalise), write
// P = softmax(S/8) as bf16 into smem in the UMMA K-major layout; O = P V is a
// 128x64x128 UMMA with V as an MN-major B operand into TMEM columns [128,192);
// O is rounded to bf16 and stored.  Rounding points match the oracle (C1.4).
__device__ __noinline__ void attention_tc(const OpDesc* op, const Ctx& X, const Smem& S, Pipe& P) {
  const MiscArgs& a = op->m;
  __nv_bfloat16* ctx = (__nv_bfloat16*)res(a.y, X);
  const int H = a.heads, units = a.N * H, HD = H * 64;
  uint8_t *sQ = S.a[0], *sK = S.a[1], *sV = S.a[2], *sP = S.b[0];
  const uint32_t tbase = *S.tmem_base;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) tma_role_fence();
  uint32_t aph = P.att_phase;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int seq = u / H, h = u - seq * H, row0 = seq * 128;
    const uint32_t ph = aph & 1;
    if (t == 0) {
      mbar_arrive_expect_tx(&S.att[0], 3 * 16384);
      tma_load_2d(smem_u32(sQ), &op->tmap_a, &S.att[0], h * 64, row0);
      tma_load_2d(smem_u32(sK), &op->tmap_a, &S.att[0], HD + h * 64, row0);
      tma_load_2d(smem_u32(sV), &op->tmap_a, &S.att[0], 2 * HD + h * 64, row0);
    }
    if (warp == 8 && lane == 0) {
      mbar_wait(&S.att[0], ph);
      tc_fence_after();
      const uint32_t idesc = umma_idesc_bf16(128, 128);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_bf16(tbase, umma_sdesc_sw128(smem_u32(sQ) + k * 32), umma_sdesc_sw128(smem_u32(sK) + k * 32), idesc,
                  k > 0 ? 1u : 0u);
      umma_commit(&S.att[1]);
    }
    if (warp >= 4 && warp < 8) {
      const int q = warp - 4, r = q * 32 + lane;
      mbar_wait(&S.att[1], ph);
      tc_fence_after();
      const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16);
      float v[32];
      float mx = -INFINITY;
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(ta + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i] * 0.125f);
      }
      float sum = 0.f;
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(ta + c * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) sum += expf(v[i] * 0.125f - mx);
      }
      const float inv = 1.f / sum;
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(ta + c * 32, v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __align__(16) __nv_bfloat16 pb[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) pb[e] = __float2bfloat16_rn(expf(v[j * 8 + e] * 0.125f - mx) * inv);
          const int chunk = (c & 1) * 4 + j;   // 16-byte chunk (8 keys) within the 64-key block
          *(uint4*)(sP + (c >> 1) * 16384 + r * 128 + ((chunk ^ (r & 7)) << 4)) = *(const uint4*)pb;
        }
      }
      fence_proxy_async_smem();
    }
    __syncthreads();
    if (warp == 8 && lane == 0) {
      tc_fence_after();
      const uint32_t idesc = umma_idesc_bf16(128, 64) | (1u << 16);   // B (V) is MN-major
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16(tbase + 128, umma_sdesc_sw128(smem_u32(sP) + (kk >> 2) * 16384 + (kk & 3) * 32),
                  umma_sdesc_sw128(smem_u32(sV) + kk * 2048), idesc, kk > 0 ? 1u : 0u);
      umma_commit(&S.att[2]);
    }
    if (warp >= 4 && warp < 8) {
      const int q = warp - 4, r = q * 32 + lane;
      mbar_wait(&S.att[2], ph);
      tc_fence_after();
      float v[32];
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tbase + ((uint32_t)(q * 32) << 16) + 128 + c * 32, v);
        __align__(16) __nv_bfloat16 ob[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) ob[i] = __float2bfloat16_rn(v[i]);
        uint4* dst = (uint4*)(ctx + (int64_t)(row0 + r) * HD + h * 64 + c * 32);
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k] = ((const uint4*)ob)[k];
      }
    }
    tc_fence_before();
    __syncthreads();
    ++aph;
  }
  if (threadIdx.x == 0) P.att_phase = aph;   // the shared pipe state (read again after a barrier)
}

// ------------------------------------------------------------------ row softmax (K11)
__device__ __noinline__ void softmax_rows(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  float* x = (float*)res(a.x, X);
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.rows; r += gridDim.x * blockDim.x) {
    float* row = x + (int64_t)r * a.cols;
    float mx = -INFINITY;
    for (int c = 0; c < a.cols; ++c) mx = fmaxf(mx, row[c]);
    float s = 0.f;
    for (int c = 0; c < a.cols; ++c) s += expf(row[c] - mx);
    const float inv = 1.f / s;
    for (int c = 0; c < a.cols; ++c) row[c] = expf(row[c] - mx) * inv;
  }
}

// ------------------------------------------------------------------ input re-layout for small-C first convs
// k = 0: 2x2 space-to-depth, y[n, P, Q, (dy*2 + dx)*C + c] = x[n, 2P+dy, 2Q+dx, c];
// k = 1: kw taps into channels, y[n, h, w, kw*C + c] = x[n, h, w + kw - pad, c]
// (zero outside the image and for the channels past KW*C).  C = 8 (one 16-B
// vector per pixel); one 16-B output vector per thread item.
__device__ __forceinline__ uint4 pack_item(const MiscArgs& a, const uint4* __restrict__ x, int i, int cv, int ov) {
  const int j = i % ov;
  int p = i / ov;
  const int w = p % a.Wo;
  p /= a.Wo;
  const int h = p % a.Ho, n = p / a.Ho;
  if (a.k == 0) {
    const int sub = j / cv, c = j % cv;   // sub = dy*2 + dx
    const int hi = 2 * h + (sub >> 1), wi = 2 * w + (sub & 1);
    return __ldcs(x + ((n * a.H + hi) * a.W + wi) * cv + c);
  }
  const int kw = j / cv, c = j % cv;
  const int wi = w + kw - a.pad;
  if (kw < a.stride && wi >= 0 && wi < a.W) return __ldg(x + ((n * a.H + h) * a.W + wi) * cv + c);
  return make_uint4(0u, 0u, 0u, 0u);
}

// Four items per thread per iteration, all loads issued before the stores
// (memory-level parallelism: the input comes from HBM).
__device__ __noinline__ void pack_input(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const uint4* x = (const uint4*)res(a.x, X);
  uint4* y = (uint4*)res(a.y, X);
  const int cv = a.C / 8;                 // input vectors per pixel
  const int ov = a.cols / 8;              // output vectors per pixel
  const int total = a.N * a.Ho * a.Wo * ov;
  const int st = gridDim.x * blockDim.x;
  for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += 4 * st) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * st < total ? pack_item(a, x, i0 + u * st, cv, ov) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * st < total) y[i0 + u * st] = v[u];
  }
}

// ------------------------------------------------------------------ 16-B vector copy
__device__ __noinline__ void copy_vec(const OpDesc* op, const Ctx& X) {
  const MiscArgs& a = op->m;
  const uint4* x = (const uint4*)res(a.x, X);
  uint4* y = (uint4*)res(a.y, X);
  const int n = a.rows, st = gridDim.x * blockDim.x;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * st < n; i += 4 * st) {
    const uint4 v0 = __ldcs(x + i), v1 = __ldcs(x + i + st), v2 = __ldcs(x + i + 2 * st), v3 = __ldcs(x + i + 3 * st);
    y[i] = v0, y[i + st] = v1, y[i + 2 * st] = v2, y[i + 3 * st] = v3;
  }
  for (; i < n; i += st) y[i] = __ldcs(x + i);
}

__device__ void run_misc(const OpDesc* op, const Ctx& X, const Smem& S, Pipe& P) {
  if (op->type == OP_ATTENTION && op->g.act_tmap) {   // qkv tensor map bound: tensor-core path
    attention_tc(op, X, S, P);
    return;
  }
  switch (op->type) {
    case OP_DWCONV: dwconv(op, X, S.scratch); break;
    case OP_MAXPOOL: maxpool(op, X); break;
    case OP_AVGPOOL: avgpool(op, X); break;
    case OP_LENET: lenet(op, X, S.scratch, S.wtag); break;
    case OP_EMBED_LN: embed_ln(op, X); break;
    case OP_LAYERNORM: layernorm(op, X); break;
    case OP_ATTENTION: attention(op, X, S.scratch); break;
    case OP_SOFTMAX: softmax_rows(op, X); break;
    case OP_SPLITK_FINAL: splitk_final(op, X); break;
    case OP_COPY: copy_vec(op, X); break;
    case OP_PACK: pack_input(op, X); break;
    default: __trap();
  }
}

__device__ void run_program(const WorkDesc& w, const Ctx& X, Smem& S, Pipe& P, ExecState* st,
                            uint64_t& epoch, uint64_t* trace, int trace_cap) {
  int i = 0, step = 0;
  const bool tr = trace && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr && trace_cap > 0) trace[0] = globaltimer();
  S.dbg = (trace && trace_cap >= 1024 + 8 * 1000) ? trace + 1024 : nullptr;
  bool staged = false;   // this step's GEMM arguments were staged during the last barrier
  int staged_j = 0;      //   and its last op (the extent was read then)
  while (i < w.n_ops) {
    // the step's extent: bound programs carry it on the step's first op (one
    // load instead of one dependent load per op of the step)
    int j = i;
    if (staged) {
      j = staged_j;
    } else {
      const int sn = w.prog[i].step_nops;
      if (sn > 0)
        j = min(w.n_ops - 1, i + sn - 1);
      else
        while (j < w.n_ops - 1 && !w.prog[j].step_end) ++j;
    }
    const int type = staged ? (int)OP_GEMM : w.prog[i].type;
    S.step = step;
    if (threadIdx.x == 0 && type != OP_LENET) *S.wtag = 0;   // smem scratch / ring reused
    const int n_next = min(kPfOps, w.n_ops - j - 1);
    prefetch_desc(w.prog + j + 1, n_next);
    const bool step_gemm = type == OP_GEMM;
    if (step_gemm) {
      gemm_step(w.prog + i, j - i + 1, X, S, P, n_next, staged);
    } else {
      if (threadIdx.x >= kThreads - 32) prefetch_ops(w.prog + j + 1, n_next, threadIdx.x - (kThreads - 32));
      for (int k = i; k <= j; ++k) run_misc(w.prog + k, X, S, P);
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 0) dbg_mark(S, 6);
    staged = false;
    bool finished = false;   // gemm_finish applied inside the barrier window
    if (w.prog[j].local_next) {
      __syncthreads();   // the next GEMM step waits per M block on completion counters
    } else {
      gridsync_arrive(st);
      // the step's counts are this CTA's own (the MMA warp wrote them before the
      // arrive's __syncthreads): thread 0 applies them before waiting
      if (step_gemm && threadIdx.x == 0) gemm_finish(P, S);
      finished = step_gemm;
      // while the other CTAs finish: the next GEMM step's arguments into shared
      // memory (read-only program data; gemm_finish's counts sit past kOpCache)
      if (j + 1 < w.n_ops && w.prog[j + 1].type == OP_GEMM) {
        const int i2 = j + 1, sn2 = w.prog[i2].step_nops;
        int j2 = i2;
        if (sn2 > 0)
          j2 = min(w.n_ops - 1, i2 + sn2 - 1);
        else
          while (j2 < w.n_ops - 1 && !w.prog[j2].step_end) ++j2;
        stage_gemm_args(w.prog + i2, j2 - i2 + 1, S);
        staged = true;
        staged_j = j2;
      }
      gridsync_wait(st, epoch, false);
    }
    if (step_gemm && !finished) {   // thread 0 applies the step's counts to the shared pipe state
      if (threadIdx.x == 0) gemm_finish(P, S);
      __syncthreads();
    }
    if (threadIdx.x == 0) dbg_mark(S, 7);
    ++step;
    if (tr && step < trace_cap) trace[step] = globaltimer();
    i = j + 1;
  }
  // every increment of this run happened before the final gpu-let barrier:
  // re-zero the counters for the next run (ordered before it by its dequeue barrier)
  const int cw = w.n_ops > 0 ? w.prog[0].cnt_words : 0;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cw; k += gridDim.x * blockDim.x) X.cnt[k] = 0u;
}

}  // namespace

extern "C" __global__ void __launch_bounds__(kThreads, 1) gl_executor(ExecParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // The CTA-uniform executor state (shared-memory layout pointers, the work
  // item's buffer bases) lives in shared memory: the interpreter's layer
  // functions take it by reference, and as stack (local-memory) objects every
  // step re-read it through L1 misses (80 % of local loads miss, ncu r6u).
  __shared__ Smem S_sh;
  __shared__ Ctx X_sh;
  Smem& S = S_sh;
  if (threadIdx.x == 0) {
  for (int s = 0; s < kStages; ++s) {
    S.a[s] = base + s * kStageBytesA;
    S.b[s] = base + kStages * kStageBytesA + s * kStageBytesB;
  }
  S.ring = base;
  uint64_t* bars = (uint64_t*)(base + kRingBytes);
  S.full = bars;                          // [kMaxStages] full, then [kMaxStages] empty
  S.empty = bars + kMaxStages;
  S.tfull = bars + 2 * kMaxStages;
  S.tempty = bars + 2 * kMaxStages + 2;
  S.att = bars + 2 * kMaxStages + 4;
  S.tmem_base = (uint32_t*)(bars + 2 * kMaxStages + 7);
  S.epi_flag = (int*)(bars + 2 * kMaxStages + 8);
  S.wtag = bars + 2 * kMaxStages + 10;
  S.estage = base + kRingBytes + 1024;
  S.scratch = base;
  S.dbg = nullptr;
  S.step = 0;
  S.tl = p.tl ? p.tl + (size_t)blockIdx.x * p.tl_cap : nullptr;
  S.tl_cap = p.tl_cap;
  S.flags = p.dbg_flags;
  S.opc = (GemmArgs*)(base + kRingBytes + 1024 + kEpiStageBytes);
  S.opn = (int*)(S.opc + kOpCache);
  S.ebias = (float*)(base + kRingBytes + 1024 + kEpiStageBytes + kOpCacheBytes);
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&S.full[s], 128 + 1);
      mbar_init(&S.empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&S.tfull[s], 1);
      mbar_init(&S.tempty[s], 8);   // one arrival per epilogue warp (count 2 each when only 4 run)
    }
    for (int s = 0; s < 3; ++s) mbar_init(&S.att[s], 1);
    *S.wtag = 0;
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc(S.tmem_base, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) {
    if (p.smid_log) p.smid_log[blockIdx.x] = (int)smid();
    p.ring->resident[blockIdx.x] = 1u;
    __threadfence_system();
  }

  // The pipe state (ring parity bits, accumulator uses, attention phase) is
  // CTA-uniform between steps: one shared copy, advanced by thread 0
  // (gemm_finish, attention_tc); each role copies it into registers.
  __shared__ __align__(16) uint8_t pipe_raw[sizeof(Pipe)];
  Pipe& P = *reinterpret_cast<Pipe*>(pipe_raw);
  if (threadIdx.x == 0) P = Pipe{};
  // barrier epochs passed: read and advanced by thread 0 only (gridsync), kept in
  // shared memory so the barrier's target is not an L1-missing stack load
  __shared__ uint64_t epoch_sh;
  if (threadIdx.x == 0) epoch_sh = 0;
  uint64_t& epoch = epoch_sh;
  int done = 0;
  // completions published so far (CTA 0 thread 0 is the only writer of the ring's completion side)
  uint64_t completions = (blockIdx.x == 0 && threadIdx.x == 0) ? p.ring->heartbeat : 0;
  for (;;) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const uint64_t head = p.st->head;
      bool quit = false;
      uint32_t ns = 64;
      for (;;) {
        if (ld_acquire_sys_u64(&p.ring->tail) > head) break;
        if (ld_acquire_sys_u64(&p.ring->quit)) {
          quit = true;
          break;
        }
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
      }
      if (quit) {
        p.st->quit = 1;
      } else {
        // the item as four 16-B loads over PCIe, ordered after the acquire of
        // `tail` above (one round trip instead of one per field)
        const uint4* src = (const uint4*)&p.ring->items[head % kRing];
        WorkDesc w;
        uint4* dst = (uint4*)&w;
        const uint4 q0 = src[0], q1 = src[1], q2 = src[2], q3 = src[3];
        dst[0] = q0, dst[1] = q1, dst[2] = q2, dst[3] = q3;
        p.st->cur = w;
        p.st->t_dequeue = globaltimer();
        p.st->head = head + 1;
      }
      __threadfence();
    }
    gridsync(p.st, epoch, true);
    if (*(volatile uint64_t*)&p.st->quit) break;
    WorkDesc w;
    {
      // the item CTA 0 broadcast, as four 16-B L2 loads (ordered after the barrier)
      const uint4* c = (const uint4*)&p.st->cur;
      uint4* dst = (uint4*)&w;
      const uint4 q0 = __ldcg(c), q1 = __ldcg(c + 1), q2 = __ldcg(c + 2), q3 = __ldcg(c + 3);
      dst[0] = q0, dst[1] = q1, dst[2] = q2, dst[3] = q3;
    }
    const uint64_t t_start = globaltimer();
    if (threadIdx.x == 0) X_sh = Ctx{(const char*)w.in, (char*)w.out, p.ws, (uint32_t*)(uintptr_t)w.prog[0].cnt_base};
    __syncthreads();
    run_program(w, X_sh, S, P, p.st, epoch, p.trace, p.trace_cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      // the record as four 16-B stores to the host-mapped ring, published by a
      // release store of comp_tail (cumulative: it also orders the batch's
      // outputs, which the final gpu-let barrier made visible to this thread)
      const uint64_t i = completions++;
      CompRec r;
      r.ticket = w.ticket;
      r.gpulet = p.gpulet;
      r.model = w.model;
      r.batch = w.batch;
      r.status = 0;
      r.t_submit_ns = w.t_submit_ns;
      r.t_dequeue_ns = p.st->t_dequeue;
      r.t_start_ns = t_start;
      r.t_end_ns = globaltimer();
      r.pad_ = 0;
      uint4* dst = (uint4*)&p.ring->comp[i % kRing];
      const uint4* srcr = (const uint4*)&r;
      dst[0] = srcr[0], dst[1] = srcr[1], dst[2] = srcr[2], dst[3] = srcr[3];
      p.ring->heartbeat = i + 1;
      st_release_sys_u64(&p.ring->comp_tail, i + 1);
    }
    if (p.one_shot > 0 && ++done >= p.one_shot) break;
  }
  __syncthreads();
  if (warp == 8) tmem_dealloc(*S.tmem_base, 512);
}

extern "C" cudaKernel_t gl_executor_handle() {
  cudaKernel_t k = nullptr;
  if (cudaGetKernel(&k, (const void*)gl_executor) != cudaSuccess) return nullptr;
  return k;
}
