"""C5 discrete-event simulator of a schedule plan (ORACLE — test infrastructure).

Arrivals (deterministic at exactly the plan rates, or Poisson with PCG64
inverse-CDF exponentials) -> per-model smooth weighted round-robin over
the model's lanes (weights = lane rates) -> per-lane FIFO with the duty-cycle
dispatch rule (C2.11: dispatch when the desired batch is formed or a
duty cycle D has passed since the window opened) -> hopeless requests dropped
((now - t_arr) + Leff(1) > SLO; drops are violations) -> the
gpu-let runs batches FIFO with Leff(b) = ceil(L(b,p) F / 1000) -> a request is
violated if t_end - t_arr > SLO.  Integer microseconds throughout.

Pinned in tests/test_oracle_des.py (Poisson mean within 3 sigma, determinism
for a fixed seed, soundness replay: deterministic arrivals at the plan rates
give 0 violations for Schedulable plans).
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
    def __init__(self, gl, m, rate, batch, F, D):
        self.gl, self.m, self.rate, self.b, self.F, self.D = gl, m, rate, batch, F, D
        self.q = []
        self.window = 0
        self.cur = 0


def simulate(plan_gpulets, prof, slo, arrivals, names=None):
    """plan_gpulets: [(size, D_us, [(m, rate, batch, F), ...]), ...];
    arrivals: {m: sorted list of int us}; returns per-model stats dict."""
    lanes, free = [], []
    by_model = {}
    for gi, (size, D, ls) in enumerate(plan_gpulets):
        free.append(0)
        for (m, rate, b, F) in ls:
            ln = Lane(gi, m, rate, b, F, D)
            ln.size = size
            lanes.append(ln)
            by_model.setdefault(m, []).append(ln)
    stats = {m: {"arrivals": 0, "late": 0, "dropped": 0, "served": 0, "lat": []} for m in arrivals}

    def leff(m, b, p, F):
        return (prof.L(m, b, p) * F + 999) // 1000

    def dispatch(ln, now):
        keep = []
        for t in ln.q:
            if (now - t) + leff(ln.m, 1, ln.size, ln.F) > slo[ln.m]:
                stats[ln.m]["dropped"] += 1
            else:
                keep.append(t)
        ln.q = keep
        ln.window = now
        if not ln.q:
            return
        k = min(len(ln.q), ln.b)
        batch, ln.q = ln.q[:k], ln.q[k:]
        start = max(now, free[ln.gl])
        end = start + leff(ln.m, k, ln.size, ln.F)
        free[ln.gl] = end
        for t in batch:
            lat = end - t
            st = stats[ln.m]
            st["served"] += 1
            st["lat"].append(lat)
            if lat > slo[ln.m]:
                st["late"] += 1

    events = []
    for m, ts in arrivals.items():
        for j, t in enumerate(ts):
            events.append((t, m, j))
        stats[m]["arrivals"] = len(ts)
    events.sort()
    timers = []          # (deadline, lane index)

    def arm(i):
        ln = lanes[i]
        if ln.q:
            heapq.heappush(timers, (ln.window + ln.D, i))

    def fire_until(t):
        while timers and timers[0][0] <= t:
            dl, i = heapq.heappop(timers)
            ln = lanes[i]
            if ln.q and ln.window + ln.D == dl:
                dispatch(ln, dl)
                arm(i)

    for t, m, _j in events:
        fire_until(t)
        cand = by_model.get(m)
        if not cand:
            stats[m]["dropped"] += 1
            continue
        total = sum(ln.rate for ln in cand)
        for ln in cand:
            ln.cur += ln.rate
        best = max(cand, key=lambda ln: ln.cur)   # first max wins ties
        best.cur -= total
        was_empty = not best.q
        best.q.append(t)
        i = lanes.index(best)
        if len(best.q) >= best.b or t - best.window >= best.D:
            dispatch(best, t)
            arm(i)
        elif was_empty:
            arm(i)
    fire_until(float("inf"))
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
