// Serving frontend (SURVEY.md §8(a) a5 + a6): replays a request-arrival trace in
// real time against live gpu-lets.  Each model's requests are routed over its
// lanes by smooth weighted round-robin (weights = the lanes' assigned rates);
// each lane keeps a FIFO and dispatches "when the desired size of request batch
// is formed or a duty-cycle is passed", after dropping
// requests that can no longer meet their SLO (drops count as violations,
// P:860).  A request's latency is host completion time - arrival time.
//
// End-to-end mode (lanes with in_host): the batch's inputs are copied from
// pinned host memory into the lane's device buffer before the batch is
// submitted, and its outputs back to the host when it completes, inside the
// measured latency; a lane then keeps one batch in flight (its device buffers
// are reused by the next batch).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <deque>
#include <unordered_map>
#include <vector>

#include "../../include/gpulet.h"

namespace {
struct LaneState {
  gl_lane cfg;
  std::deque<int64_t> q;  // request indices
  int64_t window_us = 0;
  int64_t cur = 0;        // smooth WRR credit
  bool busy = false;      // end-to-end mode: a batch of this lane is in flight
};
struct Inflight {
  int lane;
  std::vector<int64_t> reqs;
};

// Copy k request slots between a host slot array and a contiguous device buffer.
bool copy_slots(void* dev, const void* host, const std::vector<int64_t>& reqs, int64_t bytes, int32_t slots,
                bool h2d, int64_t* moved) {
  for (size_t i = 0; i < reqs.size(); ++i) {
    const int64_t slot = slots > 0 ? reqs[i] % slots : 0;
    char* d = (char*)dev + i * bytes;
    char* h = (char*)host + slot * bytes;
    const cudaError_t e = h2d ? cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, cudaStreamPerThread)
                              : cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, cudaStreamPerThread);
    if (e != cudaSuccess) return false;
    *moved += bytes;
  }
  return cudaStreamSynchronize(cudaStreamPerThread) == cudaSuccess;
}
}  // namespace

extern "C" gl_status gl_serve(gl_ctx* ctx, const gl_lane* lanes, int32_t n_lanes, int32_t n_models,
                              const int64_t* arr_us, const int32_t* arr_model, int64_t n_req, const int32_t* slo_us,
                              int64_t* lat_us, uint64_t* dev_ns, int64_t* h2d_bytes, int64_t* d2h_bytes) {
  if (!ctx || !lanes || n_lanes < 1 || n_models < 1 || (!arr_us && n_req) || !slo_us || !lat_us)
    return GL_E_ARG;
  std::vector<LaneState> L(n_lanes);
  std::vector<std::vector<int>> by_model(n_models);
  for (int i = 0; i < n_lanes; ++i) {
    L[i].cfg = lanes[i];
    if (lanes[i].model_slot < 0 || lanes[i].model_slot >= n_models) return GL_E_ARG;
    if (lanes[i].in_host && (!lanes[i].out_host || lanes[i].in_req_bytes <= 0 || lanes[i].out_req_bytes <= 0))
      return GL_E_ARG;
    by_model[lanes[i].model_slot].push_back(i);
  }
  for (int64_t r = 0; r < n_req; ++r) lat_us[r] = -2;
  int64_t h2d = 0, d2h = 0;
  uint64_t t_first = ~0ull, t_last = 0;
  std::unordered_map<uint64_t, Inflight> inflight;
  const auto t0 = std::chrono::steady_clock::now();
  auto now_us = [&] {
    return (int64_t)std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0)
        .count();
  };
  int64_t next = 0, outstanding = 0;
  gl_completion comp[128];
  const int64_t deadline = (n_req ? arr_us[n_req - 1] : 0) + 30'000'000;
  while (next < n_req || outstanding > 0) {
    const int64_t now = now_us();
    if (now > deadline) return GL_E_TIMEOUT;
    // 1. arrivals -> lanes (smooth weighted round-robin per model)
    while (next < n_req && arr_us[next] <= now) {
      const int m = arr_model[next];
      auto& cand = by_model[m];
      if (cand.empty()) {
        lat_us[next] = -1;
        ++next;
        continue;
      }
      int64_t total = 0;
      int best = -1;
      for (int li : cand) {
        L[li].cur += L[li].cfg.weight;
        total += L[li].cfg.weight;
        if (best < 0 || L[li].cur > L[best].cur) best = li;
      }
      L[best].cur -= total;
      L[best].q.push_back(next);
      ++outstanding;
      ++next;
    }
    // 2. duty-cycle dispatch
    for (int li = 0; li < n_lanes; ++li) {
      LaneState& ln = L[li];
      if (ln.q.empty() || ln.busy) continue;
      const bool full = (int)ln.q.size() >= ln.cfg.batch;
      const bool timeout = now - ln.window_us >= ln.cfg.duty_us;
      if (!full && !timeout) continue;
      while (!ln.q.empty()) {  // drop hopeless requests
        const int64_t r = ln.q.front();
        if ((now - arr_us[r]) + ln.cfg.drop_us > slo_us[arr_model[r]]) {
          lat_us[r] = -1;
          ln.q.pop_front();
          --outstanding;
        } else {
          break;
        }
      }
      ln.window_us = now;
      if (ln.q.empty()) continue;
      const int k = std::min<int>((int)ln.q.size(), ln.cfg.batch);
      std::vector<int64_t> reqs(ln.q.begin(), ln.q.begin() + k);
      if (ln.cfg.in_host &&
          !copy_slots((void*)ln.cfg.in_dev, ln.cfg.in_host, reqs, ln.cfg.in_req_bytes, ln.cfg.host_slots, true, &h2d))
        return GL_E_CUDA;
      uint64_t ticket = 0;
      const gl_status s = gl_submit_batch(ctx, ln.cfg.gpulet, ln.cfg.model_id, ln.cfg.in_dev, ln.cfg.out_dev, k,
                                          (float)slo_us[ln.cfg.model_slot] / 1000.f, &ticket);
      if (s == GL_E_QUEUE_FULL) continue;
      if (s != GL_OK) return s;
      ln.q.erase(ln.q.begin(), ln.q.begin() + k);
      ln.busy = ln.cfg.in_host != nullptr;
      inflight.emplace(ticket, Inflight{li, std::move(reqs)});
    }
    // 3. completions
    int32_t n = 0;
    const gl_status s = gl_poll(ctx, comp, 128, &n);
    if (s != GL_OK) return s;
    for (int i = 0; i < n; ++i) {
      auto it = inflight.find(comp[i].ticket);
      if (it == inflight.end()) continue;
      if (comp[i].t_dequeue_ns < t_first) t_first = comp[i].t_dequeue_ns;
      if (comp[i].t_end_ns > t_last) t_last = comp[i].t_end_ns;
      LaneState& ln = L[it->second.lane];
      if (ln.cfg.in_host) {
        if (!copy_slots(ln.cfg.out_dev, ln.cfg.out_host, it->second.reqs, ln.cfg.out_req_bytes, ln.cfg.host_slots,
                        false, &d2h))
          return GL_E_CUDA;
        ln.busy = false;
      }
      const int64_t t = now_us();
      for (int64_t r : it->second.reqs) {
        lat_us[r] = t - arr_us[r];
        --outstanding;
      }
      inflight.erase(it);
    }
  }
  if (dev_ns) {
    dev_ns[0] = t_first == ~0ull ? 0 : t_first;
    dev_ns[1] = t_last;
  }
  if (h2d_bytes) *h2d_bytes = h2d;
  if (d2h_bytes) *d2h_bytes = d2h;
  return GL_OK;
}
