// Serving frontend (SURVEY.md §8(a) a5 + a6): replays a request-arrival trace in
// real time against live gpu-lets.  Each model's requests are routed over its
// lanes by smooth weighted round-robin (weights = the lanes' assigned rates);
// each lane keeps a FIFO and dispatches "when the desired size of request batch
// is formed or a duty-cycle is passed" -- or when the batch
// it would send could otherwise no longer finish within its oldest request's SLO
// (deadline guard, DESIGN R26) -- after dropping requests that can no longer meet
// their SLO (drops count as violations).  A request's latency is
// host completion time - arrival time.
//
// The routing and dispatch rule (struct Policy) is shared with gl_serve_sim, a
// virtual-clock replay against FIFO gpu-lets whose batch sequence the tests
// compare with the discrete-event simulator oracle (oracle/des.py).
//
// End-to-end mode (lanes with in_host): a model's i-th request lives in host
// slot i % host_slots of the lane's pinned ring.  A dispatched batch goes
// through three stages, none of which blocks the frontend thread:
//   H2D  its inputs are copied into a device buffer of the lane on the lane's
//        stream (contiguous slots coalesced into one cudaMemcpyAsync), an event
//        marks the end of the copy;
//   RUN  submitted to the gpu-let once that event has completed;
//   D2H  on completion its outputs are copied back the same way; the requests
//        complete when that copy's event has completed.
// A lane has one or two device buffers (in_dev2), i.e. one or two batches in
// flight: with two, the copy of the next batch overlaps the current one's run.
// Small requests (kZeroCopyMax) skip both copies: the executor reads the
// contiguous host-ring slots of the batch and writes its outputs there itself
// (pinned memory, UVA); the bytes still cross PCIe and are counted.
#include <cuda_runtime.h>

#include <pthread.h>
#include <sched.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <deque>
#include <queue>
#include <unordered_map>
#include <vector>

#include "../../include/gpulet.h"
#include "runtime.h"

namespace {
enum Stage { FREE = 0, H2D, RUN, D2H };
// Requests at most this large (in and out) skip the copy stages: a batch of
// contiguous host-ring slots is handed to the executor as UVA-mapped pinned
// memory (LeNet 1.6 KB, BERT 512 B: a copy's fixed latency is most of their
// SLO); larger ones go through the async copy path.
constexpr int64_t kZeroCopyMax = 64 * 1024;
constexpr int kZeroCopyBuf = -2;   // Inflight::buf of a zero-copy batch

struct Batch {
  Stage stage = FREE;
  std::vector<int64_t> reqs;   // request indices
  std::vector<int64_t> slots;  // their host slots (end-to-end mode)
  cudaEvent_t ev = nullptr;
  uint64_t ticket = 0;
};

struct Inflight {
  int lane;
  int buf;                     // end-to-end buffer index; -1 plain mode, kZeroCopyBuf zero-copy batch
  std::vector<int64_t> reqs;   // plain mode: the batch's request indices
};

// ---- routing + dispatch rule (C2.11 + R26; include/gpulet.h "Dispatch rule") ------------
struct PLane {
  gl_lane cfg;
  std::deque<int64_t> q;  // request indices
  int64_t window_us = 0;  // the duty-cycle window opened at the previous dispatch
  int64_t cur = 0;        // smooth WRR credit
  int32_t leff(int k) const { return cfg.leff_us ? cfg.leff_us[k - 1] : cfg.drop_us; }
  int next_k() const { return std::min<int>((int)q.size(), cfg.batch); }
};

template <class LaneT>
struct Policy {
  std::vector<LaneT>& L;
  std::vector<std::vector<int>> by_model;
  const int64_t* arr;
  const int32_t* arr_model;
  const int32_t* slo;
  Policy(std::vector<LaneT>& L, int n_models, const int64_t* arr, const int32_t* arr_model, const int32_t* slo)
      : L(L), by_model(n_models), arr(arr), arr_model(arr_model), slo(slo) {
    for (int i = 0; i < (int)L.size(); ++i) by_model[L[i].cfg.model_slot].push_back(i);
  }
  // smooth weighted round-robin over the request's model lanes; -1: no lane serves the model
  int route(int64_t r) {
    auto& cand = by_model[arr_model[r]];
    if (cand.empty()) return -1;
    int64_t total = 0;
    int best = -1;
    for (int li : cand) {
      L[li].cur += L[li].cfg.weight;
      total += L[li].cfg.weight;
      if (best < 0 || L[li].cur > L[best].cur) best = li;
    }
    L[best].cur -= total;
    L[best].q.push_back(r);
    return best;
  }
  int32_t slo_of(const LaneT& ln) const { return slo[ln.cfg.model_slot]; }
  bool ready(int li, int64_t now) const {
    const LaneT& ln = L[li];
    if (ln.q.empty()) return false;
    if ((int)ln.q.size() >= ln.cfg.batch) return true;                    // batch formed
    if (now - ln.window_us >= ln.cfg.duty_us) return true;                // duty cycle passed
    return now - arr[ln.q.front()] + ln.leff(ln.next_k()) + ln.cfg.margin_us >= slo_of(ln);  // guard (R26, R29)
  }
  // earliest time > now at which ready() turns true with no new arrival (INT64_MAX: never)
  int64_t deadline(int li) const {
    const LaneT& ln = L[li];
    if (ln.q.empty()) return INT64_MAX;
    return std::min<int64_t>(ln.window_us + ln.cfg.duty_us,
                             arr[ln.q.front()] + slo_of(ln) - ln.leff(ln.next_k()) - ln.cfg.margin_us);
  }
  // the dispatch itself: drop hopeless requests (-> dropped), reopen the window;
  // returns the batch size k (the caller takes the k oldest from q; 0 = emptied)
  template <class F>
  int open(int li, int64_t now, F&& drop) {
    LaneT& ln = L[li];
    while (!ln.q.empty()) {
      const int64_t r = ln.q.front();
      if ((now - arr[r]) + ln.leff(1) > slo[arr_model[r]]) {
        drop(r);
        ln.q.pop_front();
      } else {
        break;
      }
    }
    ln.window_us = now;
    return ln.next_k();
  }
};

struct LaneState : PLane {
  int nbuf = 1;           // device buffers (batches in flight)
  bool zero_copy = false; // requests small enough for the executor to read / write the host ring directly
  Batch buf[2];
  cudaStream_t stream = nullptr;
  const void* in_dev(int b) const { return b ? cfg.in_dev2 : cfg.in_dev; }
  void* out_dev(int b) const { return b ? cfg.out_dev2 : cfg.out_dev; }
  int free_buf() const {
    for (int b = 0; b < nbuf; ++b)
      if (buf[b].stage == FREE) return b;
    return -1;
  }
  bool idle() const {
    for (int b = 0; b < nbuf; ++b)
      if (buf[b].stage != FREE) return false;
    return true;
  }
};

// Copy the request slots of a batch between the host ring and a contiguous
// device buffer (request i of the batch at dev + i * bytes), one async copy per
// run of consecutive slots.
bool copy_slots(void* dev, const void* host, const std::vector<int64_t>& slots, int64_t bytes, bool h2d,
                cudaStream_t st, int64_t* moved) {
  size_t i = 0;
  while (i < slots.size()) {
    size_t j = i + 1;
    while (j < slots.size() && slots[j] == slots[j - 1] + 1) ++j;
    char* d = (char*)dev + (int64_t)i * bytes;
    char* h = (char*)host + slots[i] * bytes;
    const size_t n = (j - i) * (size_t)bytes;
    const cudaError_t e = h2d ? cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, st)
                              : cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return false;
    *moved += (int64_t)n;
    i = j;
  }
  return true;
}

// Optional (gl_set_tuning(7, 1)): run the busy-polling frontend loop SCHED_FIFO
// for the duration of the call when the process may (root / CAP_SYS_NICE).  Off
// by default: measured no better than the default policy on the B200 boxes
// (profiles/ab_r1r_*.log).
struct RtGuard {
  int policy = 0;
  sched_param old{};
  bool set = false;
  RtGuard() {
    if (gl::g_tune[gl::TUNE_SERVE_RT] != 1) return;
    if (pthread_getschedparam(pthread_self(), &policy, &old) != 0) return;
    sched_param p{};
    p.sched_priority = 10;
    set = pthread_setschedparam(pthread_self(), SCHED_FIFO, &p) == 0;
  }
  ~RtGuard() {
    if (set) pthread_setschedparam(pthread_self(), policy, &old);
  }
};

struct Cleanup {
  std::vector<LaneState>& L;
  ~Cleanup() {
    for (auto& ln : L) {
      if (ln.stream) cudaStreamSynchronize(ln.stream);
      for (auto& b : ln.buf)
        if (b.ev) cudaEventDestroy(b.ev);
      if (ln.stream) cudaStreamDestroy(ln.stream);
    }
  }
};
// ---- two-stage application chains (F3, DESIGN R28) -------------------------------------------
// Requests of the trace keep indices 0..n_req-1; a completed request of model m
// creates spawn[m][m2] requests of each m2 (m2 ascending), indices in creation
// order, that reach the frontend handoff_us later and keep their root's arrival
// (deadlines, drops and latency measure from it).  Arrivals -- trace and spawned --
// are routed in (time, index) order.
struct Requests {
  std::vector<int64_t> arr;     // root arrival of every request
  std::vector<int32_t> model;
  std::vector<int32_t> parent;
  std::priority_queue<std::pair<int64_t, int64_t>, std::vector<std::pair<int64_t, int64_t>>,
                      std::greater<std::pair<int64_t, int64_t>>> pending;   // (ready time, index)
  const int32_t* spawn = nullptr;
  int32_t n_models = 0, handoff = 0;
  int64_t cap = 0;
  bool init(const int64_t* arr_us, const int32_t* arr_model, int64_t n_req, const gl_chain* ch, int32_t nm) {
    n_models = nm;
    cap = ch ? ch->cap_req : n_req;
    if (cap < n_req) return false;
    arr.reserve(cap), model.reserve(cap), parent.reserve(cap);   // data() stays valid: never grows past cap
    arr.assign(arr_us, arr_us + n_req);
    model.assign(arr_model, arr_model + n_req);
    parent.assign(n_req, -1);
    if (ch) spawn = ch->spawn, handoff = ch->handoff_us;
    return true;
  }
  // spawn the children of request r completed at t; calls made(j) for each; false: capacity
  template <class F>
  bool complete(int64_t r, int64_t t, F&& made) {
    if (!spawn) return true;
    for (int32_t m2 = 0; m2 < n_models; ++m2)
      for (int32_t c = 0; c < spawn[(int64_t)model[r] * n_models + m2]; ++c) {
        const int64_t j = (int64_t)arr.size();
        if (j >= cap) return false;
        arr.push_back(arr[r]);
        model.push_back(m2);
        parent.push_back((int32_t)r);
        pending.push({t + handoff, j});
        made(j);
      }
    return true;
  }
  // route every arrival up to t in (time, index) order
  template <class F>
  void arrivals(int64_t t, int64_t n_req, int64_t& next, F&& route) {
    for (;;) {
      const bool a = next < n_req && arr[next] <= t;
      const bool p = !pending.empty() && pending.top().first <= t;
      if (!a && !p) return;
      if (!p || (a && std::make_pair(arr[next], next) < pending.top())) {
        route(next++);
      } else {
        const int64_t j = pending.top().second;
        pending.pop();
        route(j);
      }
    }
  }
  int64_t next_time(int64_t n_req, int64_t next) const {
    int64_t t = next < n_req ? arr[next] : INT64_MAX;
    if (!pending.empty()) t = std::min(t, pending.top().first);
    return t;
  }
  void out(const gl_chain* ch_const) const {
    gl_chain* ch = const_cast<gl_chain*>(ch_const);
    if (!ch) return;
    ch->n_total = (int64_t)arr.size();
    for (size_t i = 0; i < arr.size(); ++i) {
      if (ch->parent) ch->parent[i] = parent[i];
      if (ch->req_model) ch->req_model[i] = model[i];
    }
  }
};
}  // namespace


static gl_status serve_impl(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models,
                            const int64_t* arr_us, const int32_t* arr_model, int64_t n_req, const int32_t* slo_us,
                            gl_chain* chain, int64_t* lat_us, uint64_t* dev_ns, int64_t* h2d_bytes,
                            int64_t* d2h_bytes, gl_lane_stats* lane_stats) {
  if (!ctx || !lanes || n_lanes < 1 || n_models < 1 || n_req < 0 || (!arr_us && n_req) || (!arr_model && n_req) ||
      !slo_us || !lat_us || (chain && chain->handoff_us < 0) || (chain && !chain->spawn))
    return GL_E_ARG;
  for (int64_t r = 1; r < n_req; ++r)
    if (arr_us[r] < arr_us[r - 1]) return gl::set_error(GL_E_ARG, "gl_serve: arrivals must be sorted");
  Requests R;
  if (!R.init(arr_us, arr_model, n_req, chain, n_models)) return gl::set_error(GL_E_ARG, "gl_serve: cap_req < n_req");
  std::vector<LaneState> L(n_lanes);
  Cleanup cleanup{L};
  RtGuard rt;
  for (int i = 0; i < n_lanes; ++i) {
    L[i].cfg = lanes[i];
    if (lanes[i].model_slot < 0 || lanes[i].model_slot >= n_models || lanes[i].batch < 1 || lanes[i].batch > 32 ||
        lanes[i].margin_us < 0)
      return GL_E_ARG;
    if (lanes[i].in_host) {
      if (!lanes[i].out_host || lanes[i].in_req_bytes <= 0 || lanes[i].out_req_bytes <= 0 || lanes[i].host_slots < 1)
        return GL_E_ARG;
      L[i].nbuf = (lanes[i].in_dev2 && lanes[i].out_dev2) ? 2 : 1;
      L[i].zero_copy = lanes[i].in_req_bytes <= kZeroCopyMax && lanes[i].out_req_bytes <= kZeroCopyMax;
      if (cudaStreamCreateWithFlags(&L[i].stream, cudaStreamNonBlocking) != cudaSuccess) return GL_E_CUDA;
      for (int b = 0; b < L[i].nbuf; ++b)
        if (cudaEventCreateWithFlags(&L[i].buf[b].ev, cudaEventDisableTiming) != cudaSuccess) return GL_E_CUDA;
    }
  }
  Policy<LaneState> pol(L, n_models, R.arr.data(), R.model.data(), slo_us);
  for (int64_t r = 0; r < R.cap; ++r) lat_us[r] = -2;
  if (lane_stats)
    for (int i = 0; i < n_lanes; ++i) lane_stats[i] = gl_lane_stats{0, 0, 0, 0};
  std::vector<int64_t> seq_of(R.cap, 0);   // model-local arrival index of each request (host slot rule)
  std::vector<int64_t> model_seq(n_models, 0);
  int64_t h2d = 0, d2h = 0;
  uint64_t t_first = ~0ull, t_last = 0;
  std::unordered_map<uint64_t, Inflight> inflight;
  const auto t0 = std::chrono::steady_clock::now();
  auto now_us = [&] {
    return (int64_t)std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0)
        .count();
  };
  int64_t next = 0, outstanding = 0;
  bool over_cap = false;
  // a request done at t: its latency, then its spawned successors (outstanding until served or dropped)
  auto finish = [&](int64_t r, int64_t t) {
    lat_us[r] = t - R.arr[r];
    --outstanding;
    over_cap |= !R.complete(r, t, [&](int64_t) { ++outstanding; });
  };
  auto complete = [&](Batch& b, int64_t t) {
    for (int64_t r : b.reqs) finish(r, t);
    b.reqs.clear();
    b.slots.clear();
    b.stage = FREE;
  };
  gl_completion comp[128];
  const int64_t deadline = (n_req ? arr_us[n_req - 1] : 0) + 30'000'000;
  while (next < n_req || outstanding > 0) {
    int64_t now = now_us();
    if (now > deadline) return GL_E_TIMEOUT;
    if (over_cap) return gl::set_error(GL_E_CAPACITY, "gl_serve: spawned requests exceed cap_req");
    // 1. arrivals (trace and spawned) -> lanes (smooth weighted round-robin per model)
    R.arrivals(now, n_req, next, [&](int64_t r) {
      const int m = R.model[r];
      seq_of[r] = model_seq[m]++;
      if (r < n_req) ++outstanding;   // spawned requests were counted when created
      if (pol.route(r) < 0) {
        lat_us[r] = -1;
        --outstanding;
      }
    });
    // 2. duty-cycle dispatch
    for (int li = 0; li < n_lanes; ++li) {
      LaneState& ln = L[li];
      if (ln.q.empty()) continue;
      const int b = ln.cfg.in_host ? ln.free_buf() : 0;
      if (b < 0 && !ln.zero_copy) continue;   // zero-copy batches need no device buffer
      if (!pol.ready(li, now)) continue;
      const int64_t window0 = ln.window_us;
      const int k = pol.open(li, now, [&](int64_t r) {
        lat_us[r] = -1;
        --outstanding;
      });
      if (k == 0) continue;
      if (ln.cfg.in_host) {
        std::vector<int64_t> slots(k);
        for (int i = 0; i < k; ++i) slots[i] = seq_of[ln.q[i]] % ln.cfg.host_slots;
        bool contiguous = true;
        for (int i = 1; i < k; ++i) contiguous &= slots[i] == slots[0] + i;
        if (ln.zero_copy && contiguous) {
          // small requests: the executor reads the inputs from / writes the
          // outputs to the pinned host ring itself (UVA-mapped), no copy stage
          // and no device buffer (any number of such batches in flight)
          const char* in = (const char*)ln.cfg.in_host + slots[0] * ln.cfg.in_req_bytes;
          char* out = (char*)ln.cfg.out_host + slots[0] * ln.cfg.out_req_bytes;
          uint64_t ticket = 0;
          const gl_status s = gl_submit_batch(ctx, ln.cfg.gpulet, ln.cfg.model_id, in, out, k,
                                              (float)slo_us[ln.cfg.model_slot] / 1000.f, &ticket);
          if (s == GL_E_QUEUE_FULL) continue;   // retry next iteration (the requests are still queued)
          if (s != GL_OK) return s;
          h2d += (int64_t)k * ln.cfg.in_req_bytes;
          inflight.emplace(ticket, Inflight{li, kZeroCopyBuf, std::vector<int64_t>(ln.q.begin(), ln.q.begin() + k)});
          ln.q.erase(ln.q.begin(), ln.q.begin() + k);
          continue;
        }
        if (b < 0) {                            // copy path: wait for a device buffer
          ln.window_us = window0;
          continue;
        }
        Batch& bt = ln.buf[b];
        bt.reqs.assign(ln.q.begin(), ln.q.begin() + k);
        bt.slots = std::move(slots);
        ln.q.erase(ln.q.begin(), ln.q.begin() + k);
        if (!copy_slots((void*)ln.in_dev(b), ln.cfg.in_host, bt.slots, ln.cfg.in_req_bytes, true, ln.stream, &h2d) ||
            cudaEventRecord(bt.ev, ln.stream) != cudaSuccess)
          return GL_E_CUDA;
        bt.stage = H2D;
        continue;
      }
      uint64_t ticket = 0;
      const gl_status s = gl_submit_batch(ctx, ln.cfg.gpulet, ln.cfg.model_id, ln.cfg.in_dev, ln.cfg.out_dev, k,
                                          (float)slo_us[ln.cfg.model_slot] / 1000.f, &ticket);
      if (s == GL_E_QUEUE_FULL) continue;
      if (s != GL_OK) return s;
      inflight.emplace(ticket, Inflight{li, -1, std::vector<int64_t>(ln.q.begin(), ln.q.begin() + k)});
      ln.q.erase(ln.q.begin(), ln.q.begin() + k);
    }
    // 3. end-to-end stage transitions (event polls; never block)
    for (int li = 0; li < n_lanes; ++li) {
      LaneState& ln = L[li];
      if (!ln.cfg.in_host) continue;
      for (int b = 0; b < ln.nbuf; ++b) {
        Batch& bt = ln.buf[b];
        if (bt.stage != H2D && bt.stage != D2H) continue;
        const cudaError_t q = cudaEventQuery(bt.ev);
        if (q == cudaErrorNotReady) continue;
        if (q != cudaSuccess) return GL_E_CUDA;
        if (bt.stage == D2H) {
          complete(bt, now_us());
          continue;
        }
        uint64_t ticket = 0;
        const gl_status s = gl_submit_batch(ctx, ln.cfg.gpulet, ln.cfg.model_id, ln.in_dev(b), ln.out_dev(b),
                                            (int32_t)bt.reqs.size(), (float)slo_us[ln.cfg.model_slot] / 1000.f,
                                            &ticket);
        if (s == GL_E_QUEUE_FULL) continue;
        if (s != GL_OK) return s;
        bt.ticket = ticket;
        bt.stage = RUN;
        inflight.emplace(ticket, Inflight{li, b, {}});
      }
    }
    // 4. completions
    int32_t n = 0;
    const gl_status s = gl_poll(ctx, comp, 128, &n);
    if (s != GL_OK) return s;
    for (int i = 0; i < n; ++i) {
      auto it = inflight.find(comp[i].ticket);
      if (it == inflight.end()) continue;
      if (comp[i].t_dequeue_ns < t_first) t_first = comp[i].t_dequeue_ns;
      if (comp[i].t_end_ns > t_last) t_last = comp[i].t_end_ns;
      if (lane_stats) {
        gl_lane_stats& ls = lane_stats[it->second.lane];
        ls.batches += 1;
        ls.requests += comp[i].batch;
        ls.busy_ns += comp[i].t_end_ns > comp[i].t_start_ns ? comp[i].t_end_ns - comp[i].t_start_ns : 0;
      }
      LaneState& ln = L[it->second.lane];
      const int b = it->second.buf;
      if (b < 0) {   // plain mode, or a zero-copy batch (outputs already in the host ring)
        if (b == kZeroCopyBuf) d2h += (int64_t)it->second.reqs.size() * ln.cfg.out_req_bytes;
        const int64_t t = now_us();
        for (int64_t r : it->second.reqs) finish(r, t);
        inflight.erase(it);
        continue;
      }
      inflight.erase(it);
      Batch& bt = ln.buf[b];
      if (!copy_slots(ln.out_dev(b), ln.cfg.out_host, bt.slots, ln.cfg.out_req_bytes, false, ln.stream, &d2h) ||
          cudaEventRecord(bt.ev, ln.stream) != cudaSuccess)
        return GL_E_CUDA;
      bt.stage = D2H;
    }
  }
  if (over_cap) return gl::set_error(GL_E_CAPACITY, "gl_serve: spawned requests exceed cap_req");
  if (dev_ns) {
    dev_ns[0] = t_first == ~0ull ? 0 : t_first;
    dev_ns[1] = t_last;
  }
  if (h2d_bytes) *h2d_bytes = h2d;
  if (d2h_bytes) *d2h_bytes = d2h;
  R.out(chain);
  return GL_OK;
}

extern "C" gl_status gl_serve(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models,
                              const int64_t* arr_us, const int32_t* arr_model, int64_t n_req, const int32_t* slo_us,
                              int64_t* lat_us, uint64_t* dev_ns, int64_t* h2d_bytes, int64_t* d2h_bytes,
                              gl_lane_stats* lane_stats) {
  return serve_impl(ctx, lanes, n_lanes, n_models, arr_us, arr_model, n_req, slo_us, nullptr, lat_us, dev_ns,
                    h2d_bytes, d2h_bytes, lane_stats);
}

extern "C" gl_status gl_serve_chain(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models,
                                    const int64_t* arr_us, const int32_t* arr_model, int64_t n_req,
                                    const int32_t* slo_us, gl_chain* chain, int64_t* lat_us, uint64_t* dev_ns,
                                    gl_lane_stats* lane_stats) {
  if (!chain) return gl::set_error(GL_E_ARG, "gl_serve_chain: chain is NULL");
  return serve_impl(ctx, lanes, n_lanes, n_models, arr_us, arr_model, n_req, slo_us, chain, lat_us, dev_ns, nullptr,
                    nullptr, lane_stats);
}

static gl_status serve_sim_impl(const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                                const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, gl_chain* chain,
                                int64_t* lat_us, int64_t* batch_log, int64_t cap, int64_t* n_log) {
  if (!lanes || n_lanes < 1 || n_models < 1 || (!arr_us && n_req) || (!arr_model && n_req) || !slo_us ||
      (!lat_us && n_req) || n_req < 0 || (!batch_log && cap > 0) || (chain && (chain->handoff_us < 0 || !chain->spawn)))
    return gl::set_error(GL_E_ARG, "gl_serve_sim: bad arguments");
  std::vector<PLane> L(n_lanes);
  std::unordered_map<int32_t, int64_t> free_at;   // gpu-let id -> time its FIFO drains
  for (int i = 0; i < n_lanes; ++i) {
    L[i].cfg = lanes[i];
    if (lanes[i].model_slot < 0 || lanes[i].model_slot >= n_models || !lanes[i].leff_us || lanes[i].batch < 1 ||
        lanes[i].batch > 32 || lanes[i].duty_us < 0 || lanes[i].margin_us < 0)
      return gl::set_error(GL_E_ARG, "gl_serve_sim: bad lane");
    free_at[lanes[i].gpulet] = 0;
  }
  for (int64_t r = 1; r < n_req; ++r)
    if (arr_us[r] < arr_us[r - 1]) return gl::set_error(GL_E_ARG, "gl_serve_sim: arrivals must be sorted");
  Requests R;
  if (!R.init(arr_us, arr_model, n_req, chain, n_models)) return gl::set_error(GL_E_ARG, "gl_serve_sim: cap_req < n_req");
  Policy<PLane> pol(L, n_models, R.arr.data(), R.model.data(), slo_us);
  int64_t logged = 0, next = 0;
  for (int64_t r = 0; r < R.cap; ++r) lat_us[r] = -1;
  for (;;) {
    int64_t t = R.next_time(n_req, next);
    for (int li = 0; li < n_lanes; ++li) t = std::min(t, pol.deadline(li));
    if (t == INT64_MAX) break;
    R.arrivals(t, n_req, next, [&](int64_t r) { pol.route(r); });   // no lane: stays -1 (dropped)
    for (int li = 0; li < n_lanes; ++li) {
      PLane& ln = L[li];
      while (pol.ready(li, t)) {
        const int k = pol.open(li, t, [&](int64_t r) { lat_us[r] = -1; });
        if (k == 0) break;
        int64_t& fr = free_at[ln.cfg.gpulet];
        const int64_t end = std::max(t, fr) + ln.leff(k);
        fr = end;
        if (logged < cap) {
          int64_t* row = batch_log + 4 * logged;
          row[0] = li;
          row[1] = t;
          row[2] = k;
          row[3] = ln.q.front();
        }
        ++logged;
        for (int i = 0; i < k; ++i) {
          const int64_t r = ln.q.front();
          lat_us[r] = end - R.arr[r];
          ln.q.pop_front();
          if (!R.complete(r, end, [](int64_t) {}))
            return gl::set_error(GL_E_CAPACITY, "gl_serve_sim: spawned requests exceed cap_req");
        }
      }
    }
  }
  if (n_log) *n_log = logged;
  R.out(chain);
  return GL_OK;
}

extern "C" gl_status gl_serve_sim(const gl_lane* lanes, int32_t n_lanes, int32_t n_models, const int64_t* arr_us,
                                  const int32_t* arr_model, int64_t n_req, const int32_t* slo_us, int64_t* lat_us,
                                  int64_t* batch_log, int64_t cap, int64_t* n_log) {
  return serve_sim_impl(lanes, n_lanes, n_models, arr_us, arr_model, n_req, slo_us, nullptr, lat_us, batch_log, cap,
                        n_log);
}

extern "C" gl_status gl_serve_sim_chain(const gl_lane* lanes, int32_t n_lanes, int32_t n_models,
                                        const int64_t* arr_us, const int32_t* arr_model, int64_t n_req,
                                        const int32_t* slo_us, gl_chain* chain, int64_t* lat_us, int64_t* batch_log,
                                        int64_t cap, int64_t* n_log) {
  if (!chain) return gl::set_error(GL_E_ARG, "gl_serve_sim_chain: chain is NULL");
  return serve_sim_impl(lanes, n_lanes, n_models, arr_us, arr_model, n_req, slo_us, chain, lat_us, batch_log, cap,
                        n_log);
}
