"""C5 discrete-event simulator of a schedule plan (ORACLE — test infrastructure).

Arrivals (deterministic at exactly the plan rates, or Poisson with PCG64
inverse-CDF exponentials) -> per-model smooth weighted round-robin over
the model's lanes (weights = lane rates) -> per-lane FIFO with the duty-cycle
dispatch rule (C2.11: dispatch when the desired batch is formed or a
duty cycle D has passed since the window opened; plus the deadline guard of
DESIGN R26: or when the batch it would send could otherwise not finish within
its oldest request's SLO) -> hopeless requests dropped
((now - t_arr) + Leff(1) > SLO; drops are violations) -> the
gpu-let runs batches FIFO with Leff(b) = ceil(L(b,p) F / 1000) -> a request is
violated if t_end - t_arr > SLO.  Integer microseconds throughout.

Pinned in tests/test_oracle_sched.py / tests/test_oracle_des.py (Poisson mean
within 3 sigma, determinism for a fixed seed, soundness replay: deterministic
arrivals at the plan rates give 0 violations for Schedulable plans, S:504;
hand-traced event sequences for each dispatch condition and the drop rule).
"""
import heapq
import math

import numpy as np


def arrivals_deterministic(rate, duration_us):
    if rate <= 0:
        return []
    n = (duration_us * rate) // 1_000_000
    return [(j * 1_000_000) // rate for j in range(n)]


def arrivals_poisson(rate, duration_us, seed):
    if rate <= 0:
        return []
    rng = np.random.Generator(np.random.PCG64(seed))
    out, t = [], 0.0
    while True:
        u = rng.random()
        t += -math.log(1.0 - u) / rate * 1e6
        if t >= duration_us:
            return out
        out.append(int(t))


class Lane:
    def __init__(self, gl, m, rate, batch, F, D, size, margin=0):
        self.gl, self.m, self.rate, self.b, self.F, self.D, self.size = gl, m, rate, batch, F, D, size
        self.margin = margin  # DESIGN R29: the deadline guard fires `margin` µs earlier (0: the rule as written)
        self.q = []          # request indices, oldest first
        self.window = 0      # the duty-cycle window opened at the previous dispatch
        self.cur = 0         # smooth weighted round-robin credit


def simulate_trace(plan_gpulets, prof, slo, trace, spawn=None, handoff_us=0):
    """The frontend + FIFO gpu-lets on a merged arrival trace, event by event.

    plan_gpulets: [(size, D_us, [(m, rate, batch, F), ...]), ...] (plan order);
    trace: [(t_us, m), ...] sorted by time.  Returns (lat, log): lat[i] =
    completion - arrival of request i (µs, -1 dropped / no lane), log = [(lane,
    t_dispatch, k, first request index), ...] in dispatch order.

    Rules (C2.11; DESIGN R26; include/gpulet.h "Dispatch rule"):
      * routing: each arrival goes to the lane of its model with the largest
        credit after every lane of the model gained its rate (first maximum
        wins); the chosen lane then loses the model's total rate;
      * at time t a lane with queued requests dispatches if it holds >= b
        requests, or t - window >= D, or t - arrival(oldest) + Leff(min(q, b))
        + margin >= SLO (the batch it would send could otherwise not finish in
        time; margin = the lane's jitter reserve, DESIGN R29, 0 by default);
      * a dispatch drops every queued request with (t - arrival) + Leff(1) >
        SLO, reopens the window at t, and sends the min(q, b) oldest
        requests; the lane is checked again at the same t;
      * the times considered are the arrival times and, for every lane, the
        first time its timeout or deadline condition becomes true; at each such
        time the arrivals up to it are routed first, then the lanes are
        checked in order;
      * a gpu-let runs its batches in dispatch order; a batch of k starts at
        max(t, when the gpu-let is free) and takes Leff(k) = ceil(L(k,p) F / 1000).

    Two-stage applications (F3, `traffic` P:788-790; DESIGN R28) when `spawn`
    is given ({m: [m2, ...]}): every request of model m, when its batch
    completes at `end`, creates one request of each m2 in order (indices
    len(trace), len(trace) + 1, ... in creation order) that reaches the
    frontend at end + handoff_us (the detector -> recogniser hand-off) and
    keeps its root's arrival time, so its latency, deadline-guard and drop
    tests measure from the application request's arrival against slo[m2] (the
    application's budget from its arrival).  Arrivals -- trace and spawned --
    are routed in (time, index) order.  Then returns (lat, log, parent, model)
    over all requests: parent[i] the request that spawned i (-1 for the
    trace), model[i] its model.
    """
    lanes, by_model = [], {}
    for gi, (size, D, ls) in enumerate(plan_gpulets):
        for lt in ls:   # (m, rate, b, F) or (m, rate, b, F, margin_us)
            ln = Lane(gi, *lt[:4], D, size, *lt[4:5])
            lanes.append(ln)
            by_model.setdefault(ln.m, []).append(ln)
    free = [0] * len(plan_gpulets)
    arr = [t for t, _m in trace]          # arrival of the request's root (deadlines, drops, latency)
    model = [m for _t, m in trace]
    parent = [-1] * len(trace)
    lat = [-1] * len(trace)
    log = []
    pending = []                          # spawned requests not yet routed: heap of (ready time, index)

    def leff(ln, k):
        return (prof.L(ln.m, k, ln.size) * ln.F + 999) // 1000

    def ready(ln, t):
        if not ln.q:
            return False
        k = min(len(ln.q), ln.b)
        return (len(ln.q) >= ln.b or t - ln.window >= ln.D
                or t - arr[ln.q[0]] + leff(ln, k) + ln.margin >= slo[ln.m])

    def first_ready_time(ln):
        if not ln.q:
            return None
        k = min(len(ln.q), ln.b)
        return min(ln.window + ln.D, arr[ln.q[0]] + slo[ln.m] - leff(ln, k) - ln.margin)

    def route(r):
        cand = by_model.get(model[r], [])
        if cand:
            total = sum(ln.rate for ln in cand)
            for ln in cand:
                ln.cur += ln.rate
            best = cand[0]
            for ln in cand[1:]:
                if ln.cur > best.cur:
                    best = ln
            best.cur -= total
            best.q.append(r)

    nxt = 0
    while True:
        times = [first_ready_time(ln) for ln in lanes]
        times = [x for x in times if x is not None]
        if nxt < len(trace):
            times.append(trace[nxt][0])
        if pending:
            times.append(pending[0][0])
        if not times:
            break
        t = min(times)
        while True:   # route every arrival up to t in (time, index) order
            a = (trace[nxt][0], nxt) if nxt < len(trace) and trace[nxt][0] <= t else None
            s_ = pending[0] if pending and pending[0][0] <= t else None
            if a is None and s_ is None:
                break
            if s_ is None or (a is not None and a < s_):
                route(nxt)
                nxt += 1
            else:
                heapq.heappop(pending)
                route(s_[1])
        for li, ln in enumerate(lanes):
            while ready(ln, t):
                ln.q = [r for r in ln.q if (t - arr[r]) + leff(ln, 1) <= slo[ln.m]]
                ln.window = t
                if not ln.q:
                    break
                k = min(len(ln.q), ln.b)
                batch, ln.q = ln.q[:k], ln.q[k:]
                end = max(t, free[ln.gl]) + leff(ln, k)
                free[ln.gl] = end
                log.append((li, t, k, batch[0]))
                for r in batch:
                    lat[r] = end - arr[r]
                    for m2 in (spawn or {}).get(model[r], ()):
                        arr.append(arr[r])
                        model.append(m2)
                        parent.append(r)
                        lat.append(-1)
                        heapq.heappush(pending, (end + handoff_us, len(arr) - 1))
    if spawn is None:
        return lat, log
    return lat, log, parent, model


def app_latencies(lat, parent, n_root):
    """Latency of each application request (F3): the largest latency over the
    request and its descendants (all measured from the root's arrival); -1 if
    any of them was dropped."""
    out = list(lat[:n_root])
    for i in range(n_root, len(lat)):
        r = parent[i]
        while r >= n_root:
            r = parent[r]
        if lat[i] < 0 or out[r] < 0:
            out[r] = -1
        else:
            out[r] = max(out[r], lat[i])
    return out


def simulate(plan_gpulets, prof, slo, arrivals, names=None):
    """plan_gpulets as simulate_trace; arrivals: {m: sorted list of int us} (merged by
    (time, model, index)); returns per-model stats dict."""
    trace = sorted((t, m, j) for m, ts in arrivals.items() for j, t in enumerate(ts))
    lat, _log = simulate_trace(plan_gpulets, prof, slo, [(t, m) for t, m, _j in trace])
    stats = {m: {"arrivals": len(ts), "late": 0, "dropped": 0, "served": 0, "lat": []} for m, ts in arrivals.items()}
    for (t, m, _j), x in zip(trace, lat):
        st = stats[m]
        if x < 0:
            st["dropped"] += 1
        else:
            st["served"] += 1
            st["lat"].append(x)
            if x > slo[m]:
                st["late"] += 1
    for m, st in stats.items():
        st["violations"] = st["late"] + st["dropped"]
    return stats


def plan_to_sim(plan, names):
    """oracle.sched.Plan -> simulate() input (uses the plan's dumped lane records)."""
    import json
    out = []
    for line in plan.dump.splitlines():
        d = json.loads(line)
        if "gpu" not in d or not d["lanes"]:
            continue
        out.append((d["size"], d["D_us"], [(names.index(l["model"]), l["rate"], l["batch"], l["F"])
                                            for l in d["lanes"]]))
    return out
