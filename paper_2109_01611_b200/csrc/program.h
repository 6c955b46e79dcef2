// Layer-program representation shared by the host program builder
// (models.cpp) and the device executor (executor.cu).  Plain structs only.
//
// A model is compiled, per batch size b in 1..32, into a flat array of OpDesc
// in device memory.  Ops are grouped into *steps*: the ops of one step are
// independent, their work units are spread over the gpu-let's CTAs, and a
// gpu-let-wide barrier separates steps.
#pragma once
#include <cstdint>
#include <cuda.h>

namespace gl {

enum OpType : int32_t {
  OP_GEMM = 1,         // implicit-GEMM conv / linear on tcgen05 (K1-K4)
  OP_DWCONV = 2,       // depthwise 3x3 (K5)
  OP_MAXPOOL = 3,      // k x k max pool (K6)
  OP_AVGPOOL = 4,      // global average pool (K6)
  OP_LENET = 5,        // whole LeNet-5 per image (K7)
  OP_EMBED_LN = 6,     // BERT embeddings + LayerNorm (K8)
  OP_LAYERNORM = 7,    // LayerNorm over rows (K10)
  OP_ATTENTION = 8,    // per (sequence, head) softmax(QK^T/8) V (K9)
  OP_SOFTMAX = 9,      // in-place fp32 row softmax (K11)
  OP_SPLITK_FINAL = 10, // split-K reduction epilogue
  OP_COPY = 11,        // 16-B vector copy (request input -> workspace, so TMA can read it)
  OP_PACK = 12         // request input -> workspace re-layout for small-C convs (k = 0: space-to-depth 2x2,
                       //   k = 1: the KW horizontal taps packed into channels)
};

enum BufKind : int32_t { BUF_NONE = 0, BUF_WS = 1, BUF_IN = 2, BUF_OUT = 3, BUF_ABS = 4 };
// GEMM operand sources: cp.async implicit-im2col gather by the producer warps,
// 2-D tiled TMA, or TMA im2col mode (NHWC, 64 channels x 128 pixels per load).
enum OperandSrc : int32_t { SRC_GATHER = 0, SRC_TMA = 1, SRC_IM2COL = 2 };
enum Activation : int32_t { ACT_NONE = 0, ACT_RELU = 1, ACT_GELU = 2, ACT_TANH = 3 };

struct BufRef {
  uint64_t off;   // byte offset from the base of `kind` (absolute address for BUF_ABS)
  int32_t kind;
  int32_t pad_;
};

// Operand gather geometry: rows are output pixels (n, ho, wo) of an NHWC bf16
// tensor, columns are k = (kh, kw, c) with c fastest (implicit im2col).  A plain
// [rows, K] matrix is the 1x1 case with H = W = 1 and lda = row stride.
struct Gather {
  BufRef x;
  int32_t H, W, C, lda;       // input spatial dims, channels (multiple of 8), pixel stride (elements)
  int32_t KH, KW, stride, pad;
  int32_t Ho, Wo;             // rows = n_img * Ho * Wo
  int32_t rows;               // total rows of this operand (M or N)
  int32_t padw;               // padding along W (pad is along H)
};

struct Epilogue {
  BufRef out;
  BufRef bias;                // bf16 [N] (or [M] when bias_on_m)
  BufRef res;                 // bf16 residual, same mapping as out
  BufRef ws;                  // fp32 split-K partials [splits][M][N]
  BufRef cnt;                 // int32 per-tile arrival counters (split-K last-arriver reduction)
  int64_t img_stride;         // out element index = (r / rows_per_img) * img_stride
  int32_t rows_per_img;       //   + (r % rows_per_img) * ldc + col_off + c
  int32_t ldc, col_off;
  int32_t out_fp32;           // 1: store fp32, 0: bf16
  int32_t act;
  int32_t bias_on_m;          // swap-AB: bias indexed by the A row
  int32_t transpose;          // swap-AB: (r, c) = (n, m)
  int32_t splitk;             // >1: atomically accumulate fp32 into ws
};

struct GemmArgs {
  int32_t M, N, K_real, K_pad;  // D[M,N] = A[M,K] B[N,K]^T
  int32_t BN;                   // UMMA N of this op (multiple of 16, <= 256)
  int32_t n_mblk, n_nblk, splits, kb_per_split;
  int32_t a_tma, b_tma;         // operand source: SRC_GATHER / SRC_TMA / SRC_IM2COL
  int32_t act_tmap;             // 1: the activation operand's tensor map is bound per workspace
  int32_t a_cb;                 // SRC_IM2COL channel box (64 / 32 / 16 / 8 channels per load; swizzle 128 / 64 / 32 / none)
  int32_t pad0_;
  Gather ga, gb;                // gather geometry (used when *_tma == 0)
  Epilogue ep;
  // Dataflow between GEMM steps joined without a gpu-let barrier (program.h
  // OpDesc::local_next): per-M-block completion counters (uint32 words at the
  // program's counter base; word 0 is unused, so 0 = none).
  int32_t pub_off;              // this op's counters (one per M block): each epilogue warp adds 1 per tile
  int32_t dep_a_off;            // counters of the op that wrote the A operand (wait before loading A)
  int32_t dep_r_off;            // counters of the op that wrote the residual (wait before reading it)
  int32_t dep_a_need;           // increments per producer M block once it is complete
  int32_t dep_r_need;
  int32_t dep_a_mblk;           // producer's M blocks (clamp for the im2col row range)
};

struct MiscArgs {
  BufRef x, y, w, b, g, aux;    // generic input / output / weight / bias / gamma / extra
  int32_t N, H, W, C;           // input geometry
  int32_t Ho, Wo, k, stride, pad;
  int32_t rows, cols;           // row ops (LN, softmax, split-K final)
  int32_t act;
  int32_t seq, heads, dh;       // attention
  float eps;
  int32_t pad_[2];
  Epilogue ep;                  // split-K final uses the GEMM epilogue mapping
};

struct alignas(128) OpDesc {
  CUtensorMap tmap_a;           // 128 B, 64-B aligned (TMA descriptor for A when a_tma)
  CUtensorMap tmap_b;           // (TMA descriptor for B when b_tma)
  int32_t type;
  int32_t step_end;             // 1: gpu-let barrier after this op
  int32_t n_units;              // work units (tiles) of this op
  int32_t step_nops;            // first op of a step: the step's op count (set at bind time; diagnostics)
  int32_t local_next;           // last op of a step: the next step follows with a CTA-local barrier only
                                //   (its cross-CTA inputs are covered by completion counters)
  int32_t cnt_words;            // op 0: the program's counter words (zeroed by the executor at program end)
  uint64_t cnt_base;            // op 0: device address of the counters (set when the program is uploaded)
  uint64_t pf_addr;             // read-only operand (weights) prefetched into L2 one step ahead (0: none)
  uint64_t pf_bytes;
  GemmArgs g;
  MiscArgs m;
};

// One batch of one model = one work item in a gpu-let's ring (64 B, §8(a) a6).
struct alignas(16) WorkDesc {
  uint64_t ticket;
  const OpDesc* prog;           // device program for (model, batch)
  const void* in;               // device input
  void* out;                    // device output
  int32_t n_ops;
  int32_t model;
  int32_t batch;
  int32_t slo_us;
  uint64_t t_submit_ns;         // host clock (CLOCK_MONOTONIC) at submit
  uint64_t pad_;                // 64 B: the executor reads an item as four 16-B loads
};
static_assert(sizeof(WorkDesc) == 64, "WorkDesc is one 64-B ring slot");

// Completion record (§8(a) a13): device -> host-mapped ring.
struct alignas(16) CompRec {
  uint64_t ticket;
  int32_t gpulet, model, batch, status;
  uint64_t t_submit_ns;         // host clock copied from the WorkDesc
  uint64_t t_dequeue_ns;        // %globaltimer when CTA 0 took the item
  uint64_t t_start_ns;          // after the start barrier
  uint64_t t_end_ns;            // after the last layer's barrier
  uint64_t pad_;
};
static_assert(sizeof(CompRec) == 64, "CompRec is one 64-B ring slot");

constexpr int kRing = 256;

// Host-mapped pinned region shared by the host runtime and one executor.
struct HostRing {
  volatile uint64_t tail;       // host: items published
  volatile uint64_t quit;       // host: ask the executor to exit
  volatile uint64_t resident_;  // (unused)
  volatile uint64_t error;      // device: nonzero on a detected fault
  volatile uint64_t heartbeat;  // device: items completed
  volatile uint64_t comp_tail;  // device: completions published
  uint64_t pad_[2];
  volatile uint32_t resident[160];  // device: CTA b sets resident[b] = 1 when it reaches the loop
  WorkDesc items[kRing];
  CompRec comp[kRing];
};

// Device-global executor state (one per gpu-let).
struct ExecState {
  unsigned long long barrier;   // monotonically increasing arrival counter
  uint64_t head;                // items consumed
  WorkDesc cur;                 // item broadcast by CTA 0
  uint64_t quit;
  uint64_t t_dequeue;
};

struct ExecParams {
  HostRing* ring;               // host-mapped (device pointer alias)
  ExecState* st;                // device memory
  char* ws;                     // gpu-let activation workspace
  int32_t gpulet;
  int32_t one_shot;             // >0: process this many items then exit
  int32_t* smid_log;            // optional: %smid per CTA (confinement audit)
  uint64_t* trace;              // optional: %globaltimer at program start and after every step
  int32_t trace_cap;
  int32_t dbg_flags;            // tuning experiments only (0 in production): 1 epilogue skips bias/act/stores,
                                //   2 epilogue skips global stores, 4 MMA issues no UMMA, 8 producer issues no loads,
                                //   16 MMA skips tcgen05.fence::after_thread_sync after full-barrier waits
  int32_t tl_cap;               // optional per-CTA tile timeline of step 0 (tuning tool): tl[cta * tl_cap + 4 * i + k]
  uint64_t* tl;                 //   k = 0 MMA start (accumulator acquired), 1 MMA last commit, 2 epilogue start, 3 epilogue end
};

// TMA-producer warps of a TMA-only GEMM step (warps 9 .. 8 + kTmaWarps): a thread
// that waits for a ring stage before each load sustains about one
// cp.async.bulk.tensor per ~270 ns (measured, tools/tma_micro.cu; back-to-back
// issues cost ~70 cycles each, the stage wait is the cost: tools/tma_issue_micro.cu),
// so a single producer caps a step at ~0.5 us per 64-wide K block (A + B loads);
// the producer warps take alternate K blocks.
#ifndef GL_TMA_WARPS
#define GL_TMA_WARPS 2
#endif
constexpr int kTmaWarps = GL_TMA_WARPS;
// K blocks per ring stage of a TMA-only GEMM step (executor.cu gemm_step)
#ifndef GL_KPAIR
#define GL_KPAIR 2
#endif
#ifndef GL_KPAIR_MINST
#define GL_KPAIR_MINST 3
#endif
constexpr int kKPair = GL_KPAIR;
constexpr int kKPairMinStages = GL_KPAIR_MINST;
constexpr int kThreads = 288 + 32 * kTmaWarps;   // warps 0-3 gather / epilogue, 4-7 epilogue, 8 MMA, 9.. TMA
constexpr int kStages = 4;      // fixed stage layout used as scratch by the non-GEMM ops
constexpr int kStageBytesA = 128 * 128;       // 128 rows x 64 bf16
constexpr int kStageBytesB = 256 * 128;       // up to 256 rows x 64 bf16
constexpr int kRingBytes = kStages * (kStageBytesA + kStageBytesB);  // GEMM smem ring (192 KB)
constexpr int kMaxStages = 8;   // GEMM ring depth: kRingBytes / (A + B stage bytes), at most 8
constexpr int kEpiRowBytes = 80;                   // 32 bf16 + 16 B pad per staged row
constexpr int kEpiStageBytes = 8 * 32 * kEpiRowBytes;  // 8 epilogue warps x (32 rows x 32 columns)
constexpr int kOpCache = 8;     // GEMM args of the first 8 ops of a step are cached in shared memory
constexpr int kOpCacheBytes = kOpCache * (int)sizeof(GemmArgs) + 64;
constexpr int kEpiBiasBytes = 8 * 256 * 4;        // 8 epilogue warps x up to 256 fp32 bias values of the tile
constexpr int kSmemBytes = kRingBytes + 1024 + kEpiStageBytes + kOpCacheBytes + kEpiBiasBytes;  // + barriers

}  // namespace gl
