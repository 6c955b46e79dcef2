/* gpulet.h — C-ABI of libgpulet, the B200-native gpu-let serving hot path.
 *
 * Method: arXiv 2109.01611 ("Multi-model Machine Learning Inference Serving with
 * GPU Spatial Partitioning", PAPER.md).  A gpu-let is a fraction of one GPU's
 * compute (§2.3; "up-to two virtual gpu-lets" per GPU); the
 * serving system batches requests per model and dispatches them to the gpu-let a
 * scheduler assigned (§5); the scheduler is Alg. 1 "ElasticPartitioning"
 * with the linear L2/DRAM interference model (§4.4, eq. at).
 *
 * Conventions
 *  - Plain C: no C++ or torch types cross this boundary.  All functions return a
 *    gl_status (0 = GL_OK, negative = error); gl_last_error() gives thread-local
 *    text for the last failure.
 *  - "device pointer" = a CUDA device address on the named GPU; "host pointer" =
 *    ordinary process memory.  The caller owns every pointer it passes; the
 *    library owns weights, workspaces, rings and everything behind gl_ctx.
 *  - Any CUDA error poisons the context (GL_E_CUDA on every later call).
 */
#ifndef GPULET_H
#define GPULET_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gl_ctx gl_ctx;
typedef int32_t gl_status;

enum {
  GL_OK = 0,
  GL_E_ARG = -1,            /* null pointer or bad enum */
  GL_E_GRID = -2,           /* sm_pct not in {20,40,50,60,80,100} */
  GL_E_CAPACITY = -3,       /* batch outside [1,32] */
  GL_E_PARTITION = -4,      /* sizes on one GPU sum > 100, or a third gpu-let */
  GL_E_STATE = -5,          /* submit to a destroyed gpu-let; model loaded after the gpu-let; misuse */
  GL_E_MODEL = -6,          /* model not loaded on that GPU */
  GL_E_QUEUE_FULL = -7,     /* ring full; poll and retry */
  GL_E_NOT_CONCURRENT = -8, /* executor CTAs did not all become resident (green-ctx caveat) */
  GL_E_PARSE = -9,          /* malformed weight file / input */
  GL_E_DATA = -10,          /* profile data violates monotonicity before the envelope */
  GL_E_BUDGET = -11,        /* ideal enumerator too large */
  GL_E_CUDA = -12,          /* CUDA driver/runtime error */
  GL_E_TIMEOUT = -13        /* a blocking helper exceeded its deadline */
};

/* Model kinds: the paper's five (Table tab:ml-models) + BERT-base (north_star). */
enum { GL_LENET5 = 0, GL_GOOGLENET = 1, GL_RESNET50 = 2, GL_SSD_MOBILENET_V1 = 3, GL_VGG16 = 4, GL_BERT_BASE = 5 };

/* Completion of one submitted batch.  t_submit_ns is the host
 * CLOCK_MONOTONIC at submit; the other stamps are the GPU's %globaltimer (ns):
 * dequeue = CTA 0 took the descriptor, start = all CTAs passed the start barrier,
 * end = the last layer's barrier.  Device latency = t_end_ns - t_start_ns. */
typedef struct {
  uint64_t ticket;
  int32_t gpulet, model, batch, status;
  uint64_t t_submit_ns, t_dequeue_ns, t_start_ns, t_end_ns;
} gl_completion;

/* ---- context ------------------------------------------------------------------ */
/* Open GPUs 0..num_gpus-1 (num_gpus >= 1).  Errors: GL_E_ARG, GL_E_CUDA. */
gl_status gl_init(int num_gpus, gl_ctx** out);
/* Destroy every gpu-let (draining rings), free weights.  Safe on NULL. */
gl_status gl_shutdown(gl_ctx* ctx);
/* Thread-local description of the last error (never NULL). */
const char* gl_last_error(void);

/* ---- models ------------------------------------------------------------------- */
/* Load a GLW1 weight file (written by synthgen) for model `kind` onto `gpu`:
 * repacks weights into GEMM layout, encodes TMA tensor maps and compiles the layer
 * programs for batch 1..32.  Must precede gl_create_gpulet on that GPU.
 * Out: *model_id (>= 0).  Errors: GL_E_ARG, GL_E_PARSE, GL_E_STATE, GL_E_CUDA. */
gl_status gl_load_model(gl_ctx* ctx, int gpu, int kind, const char* weight_file, int32_t* model_id);
/* Bytes of the model's input and output buffers at `batch`.  Input layouts:
 * LeNet NHWC bf16 [b,28,28,1]; GoogLeNet/ResNet-50/VGG-16 NHWC bf16 [b,224,224,8]
 * (channels 3..7 zero); SSD NHWC bf16 [b,300,300,8]; BERT int32 ids [b,128].
 * Outputs fp32: [b,classes]; SSD loc [b,3000,4] followed by conf [b,3000,21]; BERT
 * logits [b,2] followed, at byte offset roundup(8b, 16), by the pooled [CLS] vector
 * (tanh pooler output, P:741 BERT-base) bf16 [b,768]. */
gl_status gl_model_io(gl_ctx* ctx, int32_t model_id, int32_t batch, int64_t* in_bytes, int64_t* out_bytes);
/* Algorithmic FLOPs and weight bytes of one batch (for roofline accounting). */
gl_status gl_model_cost(gl_ctx* ctx, int32_t model_id, int32_t batch, double* flops, double* weight_bytes);

/* ---- gpu-lets (§2.3) ------------------------------------------- */
/* Create a gpu-let of sm_pct in {20,40,50,60,80,100} % on `gpu`: a green context
 * over SM pairs split without co-scheduling groups (the executor uses no clusters),
 * so every share is exact: 2 * round(p * SMs / 200) SMs = 30, 60, 74, 88, 118 of
 * 148 (100 % = the whole GPU, no green context), slot 0 from the front of the split
 * and slot 1 from the back (disjoint for p + q <= 100).  Drivers that refuse the
 * flag get co-scheduled 8-SM groups (never more than the share).  Runs one
 * persistent executor kernel (1 CTA per SM).  At most two per GPU, sizes summing
 * to <= 100.  Waits (<= 5 s) until every executor CTA is resident.
 * Out: *gpulet_id, *sm_count (actual SMs).  Errors: GL_E_GRID, GL_E_PARTITION,
 * GL_E_NOT_CONCURRENT, GL_E_CUDA. */
gl_status gl_create_gpulet(gl_ctx* ctx, int gpu, int sm_pct, int32_t* gpulet_id, int32_t* sm_count);
/* Create a whole GPU partition of n (1 to 4) gpu-lets, sizes pcts[] summing to <= 100,
 * in slot order.  With 3-4 gpu-lets (the paper's scheduler uses at
 * most 2) slot i takes its exact share as a contiguous range of SM pairs from the front,
 * in slot order; partitions whose exact shares exceed the GPU's SMs (20+20+20+40 %:
 * 150 > 148) are refused (GL_E_PARTITION).  All green contexts are created before the first executor starts
 * (green-context creation can block behind a running persistent kernel, so this is
 * the way to (re)partition a GPU).  The GPU must have no live gpu-let (GL_E_STATE).
 * Out: ids[n], sm_counts[n] (optional). */
gl_status gl_create_gpulets(gl_ctx* ctx, int gpu, int32_t n, const int32_t* pcts, int32_t* ids, int32_t* sm_counts);
/* The unpartitioned-concurrency baseline (Fig.
 * slo-violation "MPS(default)": concurrent kernels with no static SM partition): the same
 * executors as gl_create_gpulets, on the primary context (one non-blocking stream per
 * slot), no green context and no SM confinement -- executor i runs 2 * round(p_i * SMs /
 * 200) CTAs that the hardware block scheduler places on whatever SMs are free (one
 * executor CTA fills an SM, so the CTA counts, not SM sets, are what is fixed), with the
 * programs tiled for that CTA count.  pcts in {20,40,50,60,80}, n in {1,2}, sum <= 100;
 * gl_gpulet_smids reports where the CTAs landed.  Errors: as gl_create_gpulets. */
gl_status gl_create_gpulets_unconfined(gl_ctx* ctx, int gpu, int32_t n, const int32_t* pcts, int32_t* ids,
                                       int32_t* sm_counts);
/* Drain and stop a gpu-let's executor; its slot becomes free. */
gl_status gl_destroy_gpulet(gl_ctx* ctx, int32_t gpulet_id);
/* %smid of every executor CTA (confinement audit); *n = number written. */
gl_status gl_gpulet_smids(gl_ctx* ctx, int32_t gpulet_id, int32_t* smids, int32_t cap, int32_t* n);

/* ---- serving (§5) -------------------------------- */
/* Enqueue one batch of `model_id` on `gpulet_id` (non-blocking): writes a descriptor
 * into the gpu-let's ring.  in_dev/out_dev are device pointers on the gpu-let's GPU
 * (layouts as gl_model_io), owned by the caller and valid until the ticket is polled.
 * slo_ms is recorded for accounting only.  Out: *ticket.
 * Errors: GL_E_ARG, GL_E_CAPACITY, GL_E_MODEL, GL_E_STATE, GL_E_QUEUE_FULL. */
/* in_dev / out_dev: device memory of the gpu-let's GPU, or pinned host memory (UVA-mapped; the
 * executor reads / writes it over PCIe). */
gl_status gl_submit_batch(gl_ctx* ctx, int32_t gpulet_id, int32_t model_id, const void* in_dev, void* out_dev,
                          int32_t batch, float slo_ms, uint64_t* ticket);
/* Collect up to `max` completions across all gpu-lets (non-blocking); FIFO per
 * gpu-let.  Out: *n_out. */
gl_status gl_poll(gl_ctx* ctx, gl_completion* out, int32_t max, int32_t* n_out);
/* Block until `ticket`'s completion has been collected by gl_poll or this call
 * (timeout_ms); the record is copied to *out when non-NULL. */
gl_status gl_wait(gl_ctx* ctx, uint64_t ticket, int32_t timeout_ms, gl_completion* out);

/* ---- latency profiler (§4.3 L(b,p)) ------------------------ */
/* Run `warmup` + `reps` batches of model_id at `batch` on gpulet_id, one in flight
 * at a time, and return the median service latency as the frontend observes it:
 * gl_submit_batch -> completion visible to gl_poll (host clock, microseconds;
 * includes the ring hand-off and completion detection, which the SLO-driven
 * scheduler must budget for).  Other completions seen meanwhile are kept for
 * gl_poll. */
gl_status gl_profile(gl_ctx* ctx, int32_t gpulet_id, int32_t model_id, int32_t batch, int32_t warmup, int32_t reps,
                     const void* in_dev, void* out_dev, double* median_us);
/* gl_profile plus the q-quantile (0 <= q < 1) of the same `reps` service latencies
 * (*q_us, optional): the tail the frontend's deadline-guard margin reserves (DESIGN R29). */
gl_status gl_profile_tail(gl_ctx* ctx, int32_t gpulet_id, int32_t model_id, int32_t batch, int32_t warmup,
                          int32_t reps, const void* in_dev, void* out_dev, double q, double* median_us, double* q_us);

/* K12 HBM probe (the per-gpu-let HBM roof BW(n) is measured, not
 * assumed to be n/148 of the GPU's): a 16-B grid-stride copy of `bytes` (>= 1 MiB)
 * device buffer to another, 4 CTAs x 512 threads per SM, launched on the green
 * context of a slot-0 gpu-let of sm_pct (100 = the whole GPU); best of `reps` runs
 * after one warm-up, host-timed around a stream synchronize (use >= 256 MiB so the
 * few-µs launch/sync overhead is < 1 %).  Out: *gbs = read + write bytes / s / 1e9;
 * *sm_count (optional) = SMs it ran on.  The GPU must have no live gpu-let
 * (GL_E_STATE).  Errors: GL_E_ARG, GL_E_GRID, GL_E_STATE, GL_E_CUDA. */
gl_status gl_bw_probe(gl_ctx* ctx, int gpu, int sm_pct, int64_t bytes, int32_t reps, double* gbs, int32_t* sm_count);

/* Work-ring placement check (north_star "work queues in device memory"): the host
 * round trip of publishing one 64-B work descriptor into device memory -- an async
 * 64-B H2D copy on a non-blocking stream plus its completion -- median and p99 over
 * `reps` (>= 10) after 10 warm-up copies.  The executor's host ring (pinned, mapped)
 * needs only a host store; compare with gl_floor's whole round trip (descriptor ->
 * executor -> completion seen by the host).  Errors: GL_E_ARG, GL_E_CUDA. */
gl_status gl_publish_probe(gl_ctx* ctx, int gpu, int32_t reps, double* memcpy_us, double* memcpy_p99_us);

/* Executor floor: `warmup` + `reps` descriptors with an empty
 * program (no layer step) through gpulet_id's ring, one in flight, as gl_profile
 * measures a batch.  Out: *host_us = median submit -> completion visible to the
 * host (µs); *device_us (optional) = median start -> end stamps (the start barrier
 * and the completion write).  Needs a model loaded on the gpu-let's GPU (its
 * program pointer is carried but not run).  Errors: GL_E_ARG, GL_E_MODEL,
 * GL_E_QUEUE_FULL, GL_E_TIMEOUT. */
gl_status gl_floor(gl_ctx* ctx, int32_t gpulet_id, int32_t warmup, int32_t reps, double* host_us, double* device_us);

/* One-shot executor launch (blocking) of one batch on n_sm CTAs (whole GPU, no
 * green context): for ncu capture and per-step tracing.  trace_ns (host, cap
 * entries, optional) receives %globaltimer at program start and after each step
 * barrier; *n_steps = steps of the program. */
gl_status gl_run_once(gl_ctx* ctx, int32_t model_id, int32_t batch, const void* in_dev, void* out_dev, int32_t n_sm,
                      uint64_t* trace_ns, int32_t cap, int32_t* n_steps);
/* Per-step description of a model's layer program at `batch`: first op type, op
 * count, algorithmic FLOPs and bytes (host arrays of `cap` entries). */
gl_status gl_program_info(gl_ctx* ctx, int32_t model_id, int32_t batch, int32_t* step_type, int32_t* step_ops,
                          double* step_flops, double* step_bytes, int32_t cap, int32_t* n_steps);

/* ---- serving frontend (§5) ---------------------------- */
/* One lane of a plan: a model's share on a gpu-let (temporal sharing within it). */
typedef struct {
  int32_t gpulet;       /* gpu-let id */
  int32_t model_id;     /* loaded model id */
  int32_t model_slot;   /* index of the model in the arrival trace / slo_us */
  int32_t batch;        /* planned batch b_i (dispatch when this many are queued) */
  int32_t duty_us;      /* duty cycle D of the gpu-let (dispatch when the window is this old) */
  int32_t weight;       /* routing weight = assigned rate (smooth weighted round-robin) */
  int32_t drop_us;      /* Leff(1): a request with (now - arrival) + drop_us > SLO is dropped */
  int32_t margin_us;    /* >= 0: the deadline guard fires this much earlier (a reserve for the host /
                           PCIe jitter between the profile's median latency and a real completion;
                           DESIGN R29); 0 = the rule as written */
  const void* in_dev;   /* device input holding `batch` requests (first k used for a k-batch) */
  void* out_dev;        /* device output */
  const void* in_host;  /* NULL, or pinned host inputs (end-to-end mode): the k requests of a batch are
                           copied H2D into in_dev before it is submitted (request r of the trace uses
                           in_host + (r % host_slots) * in_req_bytes) */
  void* out_host;       /* end-to-end mode: outputs copied D2H here on completion (same slot rule) */
  int64_t in_req_bytes, out_req_bytes;  /* bytes of one request's input / output */
  int32_t host_slots;   /* requests held in in_host / out_host (per model, ring order) */
  int32_t pad2_;
  const void* in_dev2;  /* end-to-end mode, optional second device input/output pair: with it a lane keeps */
  void* out_dev2;       /*   two batches in flight (one copying while the other runs); NULL = one */
  const int32_t* leff_us; /* [32] Leff(k) = ceil(L(k, p) F / 1000) µs of this lane for k = 1..32, or NULL
                           (every k costs drop_us).  Deadline guard (DESIGN R26): a lane also dispatches
                           when (now - oldest arrival) + Leff(min(queued, batch)) >= SLO, i.e. at the
                           last moment the batch it would send can still finish in time; gl_serve_sim
                           uses it as the service time */
} gl_lane;
/* Replay an arrival trace in real time (host clock): arr_us[n_req] sorted arrival
 * times (us from the call), arr_model[n_req] model slot of each request.  Returns
 * per-request latency in lat_us (us; -1 dropped) and, when dev_ns is not NULL,
 * dev_ns[0..1] = first dequeue and last completion (%globaltimer ns) of the
 * batches it ran.  End-to-end mode (lanes with in_host): the i-th request of a
 * model (arrival order) lives in host slot i % host_slots of in_host / out_host
 * (a pinned per-model ring, as a network receive path would fill it); a batch's
 * inputs are copied H2D (asynchronously, on a per-lane stream, contiguous slots
 * coalesced into one copy) and it is submitted when the copy has landed; on
 * completion its outputs are copied D2H the same way and the requests complete
 * when that copy has landed, so the latency includes both copies.  Requests of
 * at most 64 KB in and out whose batch occupies contiguous slots skip the
 * copies: the executor reads / writes the pinned ring directly (UVA).  A lane keeps
 * one batch in flight, two with in_dev2/out_dev2.  *h2d_bytes / *d2h_bytes (may
 * be NULL) return the bytes copied; lane_stats (may be NULL; n_lanes entries) the
 * per-lane execution record.  The frontend thread never blocks on a copy
 * (gl_set_tuning(7, 1): it runs SCHED_FIFO priority 10 during the call when permitted).
 * Blocks until every request is completed or dropped.  Errors: GL_E_ARG,
 * GL_E_TIMEOUT, GL_E_CUDA, errors of submit/poll. */
/* Dispatch rule (SURVEY §8(c) C2.11 + DESIGN R26), shared by gl_serve and gl_serve_sim:
 * at time t a lane with a non-empty FIFO dispatches when (a) it holds >= batch requests,
 * (b) t - window_open >= duty_us, or (c) t - arrival(oldest) + Leff(min(queued, batch))
 * + margin_us >= SLO.  Dispatching first drops every queued request with (t - arrival) + Leff(1) > SLO
 * (a drop is a violation), reopens the window at t and sends the
 * min(queued, batch) oldest requests.  Arrivals are routed (smooth weighted round-robin
 * over the model's lanes, weights = assigned rates, first maximum wins) before the lanes
 * are checked in lane order; a lane re-checks at the same t after a dispatch. */

/* Virtual-clock replay of the same frontend (no GPU; the fake backend of SURVEY §8(c)
 * C5): the dispatch rule above, evaluated at every arrival and at every lane deadline
 * (window_open + duty_us, arrival(oldest) + SLO - Leff(min(queued, batch))), against
 * gpu-lets that run their batches FIFO, each taking Leff(k) of its lane (leff_us must
 * be set).  Lanes with the same `gpulet` id share one FIFO.  Only the lane fields
 * gpulet, model_slot, batch, duty_us, weight, drop_us, leff_us are read.  Out:
 * lat_us[n_req] = completion - arrival (µs; -1 dropped or no lane for the model);
 * batch_log (optional, cap rows of 4 int64: lane, dispatch time, k, index of the
 * batch's first request in the trace) and *n_log (rows produced; rows past cap are
 * counted, not written).  Errors: GL_E_ARG. */
gl_status gl_serve_sim(const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                       const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, int64_t* lat_us,
                       int64_t* batch_log, int64_t cap, int64_t* n_log);

/* Per-lane execution record of one gl_serve call: batches and requests run, and
 * the summed device time of its batches (t_end - t_start, %globaltimer ns: the
 * executor's own clock, since a persistent kernel has no per-batch launch). */
typedef struct {
  int64_t batches;
  int64_t requests;
  uint64_t busy_ns;
  uint64_t pad_;
} gl_lane_stats;
gl_status gl_serve(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                   const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, int64_t* lat_us,
                   uint64_t* dev_ns, int64_t* h2d_bytes, int64_t* d2h_bytes, gl_lane_stats* lane_stats);

/* Two-stage applications (`traffic` P:788-790: SSD-MobileNet detects,
 * GoogLeNet and VGG-16 recognise; DESIGN R28).  A request of model i, when its batch
 * completes at t, creates spawn[i * n_models + j] requests of each model j (j ascending;
 * indices n_req, n_req + 1, ... in creation order) that reach the frontend at
 * t + handoff_us (the detector -> recogniser hand-off: box decode, NMS and crops, see
 * gl_ssd_detect / gl_crop_resize) and keep the arrival time of the trace request they
 * descend from: their latency, deadline guard and drop test are measured from it
 * against slo_us[j] (the application's budget from its arrival), so the stage split of
 * an application SLO is expressed by the SLOs of its first-stage models.  Trace and
 * spawned arrivals are routed in (time, index) order.  A dropped request spawns nothing;
 * a late one still does.  lat_us / parent / req_model hold cap_req entries (trace +
 * spawned); GL_E_CAPACITY if a run would create more. */
typedef struct {
  const int32_t* spawn;      /* [n_models][n_models] requests created per completion */
  int32_t handoff_us;        /* >= 0 */
  int32_t pad_;
  int64_t cap_req;           /* >= n_req: capacity of lat_us, parent, req_model */
  int32_t* parent;           /* out (optional): spawning request, -1 for trace requests */
  int32_t* req_model;        /* out (optional): model slot of every request */
  int64_t n_total;           /* out: requests of the run (trace + spawned) */
} gl_chain;
/* gl_serve with application chains (plain or end-to-end lanes as gl_serve; a spawned
 * request of model j takes the next host slot of model j in end-to-end mode). */
gl_status gl_serve_chain(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                         const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, gl_chain* chain,
                         int64_t* lat_us, uint64_t* dev_ns, gl_lane_stats* lane_stats);
/* gl_serve_sim with application chains: a completion is the end of its batch on the
 * virtual FIFO gpu-let (oracle: oracle/des.py simulate_trace(spawn=...)). */
gl_status gl_serve_sim_chain(const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                             const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, gl_chain* chain,
                             int64_t* lat_us, int64_t* batch_log, int64_t cap, int64_t* n_log);

/* ---- scheduler (Alg. 1) --------------------------------- */
typedef struct {
  int32_t n_models;          /* <= 8, canonical order */
  const char* const* names;  /* model names printed in the plan */
  const int32_t* lat_us;     /* L(b,p): [n_models][32][6], p in {20,40,50,60,80,100} */
  const double* l2;          /* solo L2 util: [n_models][6 stat batches 1,2,4,8,16,32][6] */
  const double* mem;         /* solo DRAM util: same shape */
  const int32_t* slo_us;     /* [n_models] */
  const int32_t* rates;      /* [n_models] req/s */
  double coeffs[5];          /* c1..c5 of P:641 (used by mode 1) */
  int32_t num_gpus;
  int32_t mode;              /* 0 gpulet, 1 gpulet+int, 2 sbp (whole-GPU temporal), 3 ideal, 4 sbp50 (SBP on
                                the two 50 % gpu-lets of every GPU, Fig. success-case) */
  const int32_t* sm_count;   /* [6] SMs of each grid size (printed as "sm" in the plan dump); NULL = the
                                exact shares of 148 SMs in SM pairs: 30, 60, 74, 88, 118, 148 */
} gl_sched_input;
/* Array form of the scheduler (callers that already hold the tables, e.g. the
 * scheduler sweeps).  Produce the canonical plan dump (JSON lines)
 * into plan_buf (cap bytes, NUL-terminated); *len = bytes written (excluding
 * NUL); *verdict = 1 Schedulable / 0 NotSchedulable.  Integer maths except the
 * knee and the factor (IEEE double, fixed order).  Errors: GL_E_ARG, GL_E_BUDGET
 * (buffer too small). */
gl_status gl_schedule(const gl_sched_input* in, char* plan_buf, size_t cap, size_t* len, int32_t* verdict);

/* ---- SPEC-format files: profile CSV, coeffs JSON, workload JSON ------
 * Profile CSV (SPEC S:130 + sm_count): header row naming at least
 *   model,batch,partition_pct and latency_us (integer or decimal µs) or latency_ms
 *   (decimal ms, SPEC's unit); optional sm_count, l2_util, mem_bw_util (blank allowed;
 *   read at the stat batches 1,2,4,8,16,32 only).  Decimal latencies are converted
 *   exactly (decimal shift) and rounded UP to whole µs.  Every one of the
 *   six canonical models (lenet5, googlenet, resnet50, ssd_mobilenet_v1, vgg16,
 *   bert_base) needs all 32 x 6 (batch 1..32, p in {20,40,50,60,80,100}) rows.
 * C4.1: unless `flags` bit 0 (strict, SPEC S:41-42 / S:58) is set the
 *   latencies are replaced by their min-envelope L*(b,p) = min over b' >= b, p' <= p
 *   (realisable: pad the batch / run on fewer SMs); strict mode keeps the raw table
 *   and reports a monotonicity violation as GL_E_DATA.
 * Errors: GL_E_ARG (NULL), GL_E_PARSE (unreadable file, malformed row: gl_last_error
 *   names the line), GL_E_DATA (unknown model, p off the grid, batch outside 1..32,
 *   duplicate or missing row, latency <= 0, utilisation outside [0,1], inconsistent
 *   sm_count, strict-mode monotonicity violation naming (model, b, p)).
 * Out (host arrays, all optional): lat_us [6][32][6] int µs; l2, mem [6][6 stat
 *   batches][6] doubles (0 where blank); sm_count [6] (from the CSV, else the defaults
 *   of gl_sched_input). */
gl_status gl_profile_load(const char* profile_csv, int32_t flags, int32_t* lat_us, double* l2, double* mem,
                          int32_t* sm_count);

/* SLOs and rates of a workload from an enveloped table
 * lat_us [6][32][6]:
 *  slo_mode 0 = rule: SLO_m = 2 * L*_m(32, 100 %) ("set by doubling the
 *    solo execution latency ... batch size of 32"); 1 = table: Table tab:ml-models
 *    constants (goo 44, le 5, res 95, ssd 136, vgg 130 ms; BERT 95 ms).
 *  scenario (C4.4): "equal"/"mix6" (50 x 6), "long-only" (0,0,100,100,100,100),
 *    "short-skew" (100,100,100,50,50,50), "game" (app rate 100 -> 600 LeNet + 100
 *    ResNet-50), "traffic" (100 SSD + 100 GoogLeNet + 100 VGG-16).
 *  rate_m = floor(((double)(base_m * SLO_paper_ref_us) * x) / (double)SLO_ref_us) * num_gpus
 *    in IEEE double, this order (C4.3: the B200 time compression; ref = the model
 *    itself, ResNet-50 for BERT; for game / traffic one scale for the whole app, its
 *    app-SLO model's: ResNet-50 / SSD, DESIGN R23).  In table mode the scale is 1.
 * Out: slo_us[6], rates[6].  Errors: GL_E_ARG (NULL, unknown scenario or slo_mode,
 *   x < 0 or not finite, num_gpus < 1). */
gl_status gl_workload_rates(const int32_t* lat_us, int32_t slo_mode, const char* scenario, double x,
                            int32_t num_gpus, int32_t* slo_us, int32_t* rates);

/* The scheduler driven by files (SPEC S:130 profile, S:346 workload,
 * S:272 plan dump).  profile_csv: a path.  coeffs_json: a path or inline JSON text
 * (first non-blank character '{') holding "coeffs": [c1..c5]; NULL = no
 * interference model (only mode gpulet+int needs it).  workload_json: a path or inline
 * JSON object with
 *   "num_gpus": N (default 1), "mode": "gpulet" | "gpulet+int" | "sbp" | "ideal" | "sbp50",
 *   "slo_mode": "rule" (default) | "table", "envelope": true (default) | false (strict),
 *   and the rates as one of
 *     "scenario": name + optional "x" (multiplier, default 1.0)  -> gl_workload_rates;
 *     "base_rates": [6 ints] paper-scale rates + optional "x": scaled per model as a
 *       non-application scenario of gl_workload_rates (the paper's sweep);
 *     "rates": [6 ints] (total req/s, canonical order);
 *     "models": [{"name", "rate", optional "slo_ms"}]  (SPEC S:346 form; models not
 *       listed get rate 0; slo_ms overrides the slo_mode SLO, rounded up to µs).
 * Output (plan_buf, cap bytes, NUL-terminated, *len without the NUL): a header line
 *   {"slo_us":[..],"rates":[..],"num_gpus":N,"mode":"..","slo_mode":".."}
 * followed by gl_schedule's canonical plan dump with the profile's sm_count.  In
 * scenario / base_rates form a model whose base rate is positive but whose scaled rate truncates
 * to 0 makes the workload NotSchedulable without running the scheduler (header +
 * {"verdict":"NotSchedulable","failed_model":name,"reason":"rate_truncated"}): the
 * scenario's composition would be lost.  *verdict = 1 Schedulable / 0 not.
 * Errors: those of gl_profile_load; GL_E_PARSE (malformed JSON: gl_last_error names the
 *   offset), GL_E_ARG (bad field value), GL_E_BUDGET (buffer too small). */
gl_status gl_schedule_files(const char* profile_csv, const char* coeffs_json, const char* workload_json,
                            char* plan_buf, size_t cap, size_t* len, int32_t* verdict);
/* Ordinary least squares for the interference model (§4.4): X [n][5] row-major,
 * y [n]; out c[5].  Householder QR.  Errors: GL_E_ARG, GL_E_DATA (rank < 5). */
gl_status gl_fit_interference(const double* X, const double* y, int32_t n, double* c);

/* ---- kernel unit entry points (tests; one-shot executor on the whole GPU) ------------ */
/* D[M,N] = A[M,K] W[N,K]^T + bias -> act; A, out device pointers (A bf16 [M,K]); W, bias
 * HOST bf16 bits.  act: 0 none 1 relu 2 gelu 3 tanh.  swap_ab: weights as the UMMA M
 * operand (small M).  splitk: allow split-K.  a_in_ws: copy A into the executor
 * workspace first so the TMA operand path (bound tensor map) is exercised. */
gl_status gl_test_gemm(gl_ctx* ctx, int gpu, const void* A_dev, const uint16_t* W_host, const uint16_t* bias_host,
                       void* out_dev, int32_t M, int32_t N, int32_t K, int32_t act, int32_t swap_ab, int32_t splitk,
                       int32_t out_fp32, int32_t a_in_ws);
/* Conv (NHWC bf16 x [N,H,W,C], C % 8 == 0; W host OHWI [Cout,KH,KH,C]) + bias + act -> y.
 * x_in_ws: stage x in the workspace (TMA 2-D / im2col operand paths). */
gl_status gl_test_conv(gl_ctx* ctx, int gpu, const void* x_dev, const uint16_t* W_host, const uint16_t* bias_host,
                       void* y_dev, int32_t N, int32_t H, int32_t W, int32_t C, int32_t Cout, int32_t KH,
                       int32_t stride, int32_t pad, int32_t act, int32_t x_in_ws);
/* Misc CUDA-core op (type = executor op id: 2 dwconv, 3 maxpool, 4 avgpool, 7 layernorm,
 * 8 attention, 9 softmax) with integer args `iargs` and host bf16 params. */
gl_status gl_test_misc(gl_ctx* ctx, int gpu, int32_t type, const int32_t* iargs, int32_t n_iargs,
                       const uint16_t* params_host, int64_t n_params, const void* x_dev, void* y_dev);

/* Statistics of the last kernel-unit test run (gl_test_gemm/conv/misc launch the
 * one-op program once, after gl_set_tuning(3, n) warm-up launches): *ns = measured device duration
 * (%globaltimer, program start -> final barrier); timeline (host buffer, `cap`
 * uint64) = per-CTA tile stamps of the GEMM step, `*tl_per_cta` entries per CTA,
 * entry 4*i+k of CTA c at [c * tl_per_cta + 4*i + k], k = 0 MMA start, 1 MMA last
 * commit, 2 epilogue start, 3 epilogue end, ns from program start (0 = unused).
 * Any pointer may be NULL.  Process-global; not thread-safe (a tuning tool). */
gl_status gl_test_stats(uint64_t* ns, uint64_t* timeline, int32_t cap, int32_t* tl_per_cta);

/* Program-builder tuning overrides for models loaded / tests built afterwards
 * (process-global; 0 = automatic).  key 0: GEMM UMMA N tile (BN, multiple of 16,
 * <= 256); key 1: split-K factor (1 = off); key 2: executor debug flags (tuning
 * experiments, see ExecParams::dbg_flags); key 3: warm-up launches of the kernel-unit
 * tests; key 4: 1 = gather every activation operand with cp.async (no TMA), to
 * test that path; key 5: SM count the programs are tiled for (>= 8); key 6: 1 =
 * barrier-free GEMM step joins, 2 = also log the plan to stderr; key 7:
 * 1 = gl_serve polls SCHED_FIFO when the process may.  GL_E_ARG for an unknown key. */
gl_status gl_set_tuning(int32_t key, int32_t value);

/* ---- F3: the `traffic` application's detection -> recognition hand-off ----
 * PAPER.md P:788-790 ("traffic": SSD-MobileNet detects objects, GoogLeNet and
 * VGG-16 recognise them) and SURVEY §8(f) F3.  The paper does not define the
 * detector's output stage; these calls implement the textbook SSD one with the
 * readings of DESIGN.md §2 R27 (priors, variances 0.1/0.2, per-class greedy
 * NMS, merge order, half-pixel bilinear crops).  They are stand-alone stream
 * kernels (no gl_ctx): every pointer is a device pointer on the current
 * device, owned by the caller; the calls are asynchronous on `stream` (a
 * cudaStream_t, NULL = legacy default stream).  GL_E_ARG (with
 * gl_last_error text) for a bad size or NULL pointer, GL_E_CUDA if a launch
 * fails.  n_img == 0 is a no-op. */

/* Workspace bytes gl_ssd_detect needs for n_img images and top_k (1..400). */
gl_status gl_ssd_detect_workspace(int32_t n_img, int32_t top_k, size_t* bytes);

/* SSD post-processing of the ssd_mobilenet_v1 model output (its layout,
 * gl_model_io): loc [n_img][3000][4] fp32 (offsets per prior, head order map,
 * row, column, prior) and conf [n_img][3000][21] fp32 softmax scores (class 0 =
 * background).  Per image and class 1..20: priors with score > score_thr,
 * ordered by (score desc, prior asc), the first top_k decoded and greedily
 * suppressed (IoU > iou_thr, fp32); then all classes' survivors ordered by
 * (score desc, class asc, prior asc), the first max_det written to det
 * [n_img][max_det][7] = (x1, y1, x2, y2 in [0, 1], score, class, prior) and
 * their number to count [n_img].  Rows past count are left untouched. */
gl_status gl_ssd_detect(const float* loc_dev, const float* conf_dev, int32_t n_img, float score_thr, float iou_thr,
                        int32_t top_k, int32_t max_det, float* det_dev, int32_t* count_dev, void* ws_dev,
                        size_t ws_bytes, void* stream);

/* Crops for the recognisers: for image n and slot k < per_img, detection k of
 * gl_ssd_detect's output (det/count/max_det as written there) is cut from img
 * [n_img][H][W][C] bf16 (NHWC, C == 8: the models' padded input layout) and
 * resized to [OH][OW][C] by bilinear sampling with half-pixel centres (R27),
 * written to out [n_img * per_img][OH][OW][C] bf16 at crop n * per_img + k;
 * slots k >= count[n] are zero-filled. */
gl_status gl_crop_resize(const void* img_dev, int32_t n_img, int32_t H, int32_t W, int32_t C, const float* det_dev,
                         const int32_t* count_dev, int32_t max_det, int32_t per_img, int32_t OH, int32_t OW,
                         void* out_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GPULET_H */
