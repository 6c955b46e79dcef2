"""C2 scheduler oracle (ORACLE — test infrastructure only).

Step-by-step restatement of the paper's Algorithm 1 (ElasticPartitioning +
FindBestFit, text P:566-598) under the readings of
SURVEY.md §8(c) C2 (listed in DESIGN.md §2), plus the SBP whole-GPU temporal
baseline (reading C2.9) and the ideal / brute-force enumerators
(C2.10).

Units (C2.1): latencies and SLOs are int microseconds, rates int req/s,
interference factor F int per-mille (>= 1000), sizes int percent.  All
rate/capacity comparisons are exact int cross-multiplications.  Only the knee
(C2.4) and the factor (C2.7) use IEEE double, in the operation order written
below (the C++ scheduler must reproduce plans byte for byte, C2.12).

Pins: tests/test_oracle_sched.py (SPEC worked examples S:80-S:310, SURVEY W1-W3,
SLO rule invariant, invariants after every step, brute force on tiny instances,
soundness replay through the DES).
"""
import json
import math
from dataclasses import dataclass, field
from itertools import combinations_with_replacement, product

GRID = (20, 40, 50, 60, 80, 100)
# exact shares of 148 SMs in SM pairs (DESIGN R15); a Profile may carry measured counts
SM_OF = {20: 30, 40: 60, 50: 74, 60: 88, 80: 118, 100: 148}
BMAX = 32
STAT_B = (1, 2, 4, 8, 16, 32)
EPS_KNEE = 1e-9
MODES = ("gpulet", "gpulet+int", "sbp", "sbp50")


class Profile:
    """L(b,p) in int us for b in 1..32, p in GRID; solo stats l2/mem at STAT_B.

    lat[m][b-1][gi], l2[m][si][gi], mem[m][si][gi]; models are indices into
    `names` (canonical order le, goo, res, ssd, vgg, bert — C6 #22)."""

    def __init__(self, names, lat, l2=None, mem=None, sm=None):
        self.names = list(names)
        self.sm = dict(zip(GRID, sm)) if sm is not None else dict(SM_OF)
        self.lat = lat
        M = len(names)
        self.l2 = l2 if l2 is not None else [[[0.0] * 6 for _ in STAT_B] for _ in range(M)]
        self.mem = mem if mem is not None else [[[0.0] * 6 for _ in STAT_B] for _ in range(M)]

    def L(self, m, b, p):
        return self.lat[m][b - 1][GRID.index(p)]

    def stat_index(self, b):
        """Smallest measured stat batch >= b (S:67 ceiling rule)."""
        for i, sb in enumerate(STAT_B):
            if sb >= b:
                return i
        raise ValueError(b)

    def l2_at(self, m, b, p):
        return self.l2[m][self.stat_index(b)][GRID.index(p)]

    def mem_at(self, m, b, p):
        return self.mem[m][self.stat_index(b)][GRID.index(p)]


@dataclass
class Lane:
    m: int
    r: int


@dataclass
class Gpulet:
    gpu: int
    slot: int
    size: int
    lanes: list = field(default_factory=list)

    def key(self):
        return (self.gpu, self.slot)


class Scheduler:
    """One scheduling decision (one period of Alg. 1's outer loop)."""

    def __init__(self, prof, slo, coeffs, mode):
        assert mode in MODES
        self.P, self.slo, self.c, self.mode = prof, list(slo), coeffs, mode
        self.use_int = mode == "gpulet+int"

    # ---- C2.2 effective latency, max batch, capacity -----------------------
    def leff(self, m, b, p, F):
        return (self.P.L(m, b, p) * F + 999) // 1000

    def b_sat(self, m, p):
        """max{b : 2 L(b,p) <= SLO_m} (duty-cycle rule, C6 #7), None if none."""
        best = None
        for b in range(1, BMAX + 1):
            if 2 * self.P.L(m, b, p) <= self.slo[m]:
                best = b
        return best

    def b_int(self, m, p, A):
        """Interference-aware batch (reading R13, P:532-537 / P:594: "the maximum
        batch size b is decided and checked whether it can meet the SLO when there
        is the additional interference-induced overhead"): the largest b <= b_sat
        with 2 Leff(b, F(b)) <= SLO_m, or None.  Equals b_sat without interference."""
        b0 = self.b_sat(m, p)
        if b0 is None:
            return None
        for b in range(b0, 0, -1):
            if 2 * self.leff(m, b, p, self.factor(m, b, p, A)) <= self.slo[m]:
                return b
        return None

    def cap(self, m, p, F=1000):
        b = self.b_sat(m, p)
        if b is None:
            return 0
        return b * 1_000_000 // self.leff(m, b, p, F)

    # ---- C2.3 capacity curve, C2.4 knee, C2.5 p_req ------------------------
    def curve(self, m):
        out = []
        for p in GRID:
            best = 0
            for b in range(1, BMAX + 1):
                L = self.P.L(m, b, p)
                if 2 * L <= self.slo[m]:
                    best = max(best, b * 1_000_000 // L)
            out.append(best)
        return out

    def p_eff(self, m):
        """MaxEfficientPartition: knee = max curvature of the
        normalised rate-vs-size curve; None if the model is infeasible."""
        return knee(self.curve(m))

    def p_req(self, m, R):
        """MinRequiredPartition: smallest p with r(p) >= R, else 100."""
        for p, r in zip(GRID, self.curve(m)):
            if r >= R:
                return p
        return 100

    # ---- C2.7 interference factor ------------------------------------------
    def aggregate(self, h):
        """Partner aggregate A(h) = (max l2, max mem) over h's lanes at (batch, h.size)."""
        if h is None or not h.lanes:
            return None
        recs = self.eval_lanes(h, None, check_only_batches=True)
        l2 = max(self.P.l2_at(ln.m, b, h.size) for ln, b in recs)
        mem = max(self.P.mem_at(ln.m, b, h.size) for ln, b in recs)
        return (l2, mem)

    def factor(self, m, b, p, A):
        if not self.use_int or A is None:
            return 1000
        c1, c2, c3, c4, c5 = self.c
        raw = ((((c1 * self.P.l2_at(m, b, p)) + (c2 * A[0])) + (c3 * self.P.mem_at(m, b, p)))
               + (c4 * A[1])) + c5
        return max(1000, math.ceil(1000.0 * raw))

    # ---- C2.6 lane-set feasibility ------------------------------------------
    def eval_lanes(self, g, A, check_only_batches=False, lanes=None, size=None):
        """Evaluate a lane set on gpu-let g (size p) under partner aggregate A.

        Returns (D, [(lane, b, e, F)]) if feasible else None.  With
        check_only_batches=True returns [(lane, b)] (interference-free batches,
        used to look up the stats that form A(g))."""
        lanes = g.lanes if lanes is None else lanes
        p = g.size if size is None else size
        if len(lanes) == 1:
            ln = lanes[0]
            if check_only_batches:        # stats lookup only: never fails
                return [(ln, self.b_sat(ln.m, p) or 1)]
            b = self.b_int(ln.m, p, A)
            if b is None:
                return None
            F = self.factor(ln.m, b, p, A)
            e = self.leff(ln.m, b, p, F)
            if 2 * e > self.slo[ln.m] or ln.r * e > b * 1_000_000:
                return None
            return (e, [(ln, b, e, F)])
        # k >= 2 lanes: Nexus-style merge
        Ds = []
        for ln in lanes:
            b = self.b_sat(ln.m, p) if check_only_batches else self.b_int(ln.m, p, A)
            if b is None:
                if check_only_batches:
                    return [(l2, 1) for l2 in lanes]
                return None
            F = 1000 if check_only_batches else self.factor(ln.m, b, p, A)
            Ds.append(self.leff(ln.m, b, p, F))
        D = min(Ds)
        recs, tot = [], 0
        for ln in lanes:
            b = max(1, (ln.r * D + 999_999) // 1_000_000)
            if check_only_batches:
                recs.append((ln, min(b, BMAX)))
                continue
            if b > BMAX:
                return None
            F = self.factor(ln.m, b, p, A)
            e = self.leff(ln.m, b, p, F)
            tot += e
            recs.append((ln, b, e, F))
        if check_only_batches:
            return recs
        # sum(e) <= D (the round fits the duty cycle) and, per lane, batch
        # building D + the whole round sum(e) <= SLO_i (reading C6 #18, S:243;
        # worst case under FIFO round-based execution)
        if tot > D or any(D + tot > self.slo[ln.m] for ln, _b, _e, _F in recs):
            return None
        return (D, recs)

    # ---- inventory helpers ----------------------------------------------------
    def sibling(self, g):
        for h in self.remain + self.alloc:
            if h.gpu == g.gpu and h.slot != g.slot:
                return h
        return None

    def feasible(self, g, lanes=None, sib_override=None):
        sib = self.sibling(g) if sib_override is None else sib_override
        return self.eval_lanes(g, self.aggregate(sib), lanes=lanes) is not None

    def sibling_ok(self, g):
        """Sibling re-check (C2.7): g's sibling must stay feasible under A(g)."""
        h = self.sibling(g)
        if h is None or not h.lanes:
            return True
        return self.eval_lanes(h, self.aggregate(g)) is not None

    # ---- C2.8 ElasticPartitioning / FindBestFit (Alg. 1) -----------------------
    def run(self, rates, num_gpus, layout=None):
        """Alg. 1 for one period. layout=None -> elastic (Split/RevertSplit);
        layout=[sizes per gpu] -> fixed layout (ideal, C2.10)."""
        self.fixed = layout is not None
        if layout is None:
            self.remain = [Gpulet(i, 0, 100) for i in range(num_gpus)]
        else:
            self.remain = []
            for i, sizes in enumerate(layout):
                for s, sz in enumerate(sizes):
                    self.remain.append(Gpulet(i, s, sz))
        self.alloc = []
        order = sorted([m for m in range(len(rates)) if rates[m] > 0], key=lambda m: (-rates[m], m))
        for m in order:
            pe = self.p_eff(m)
            if pe is None:
                return self.result(False, m)
            R = rates[m]
            while R > 0:
                p_ideal = min(pe, self.p_req(m, R))
                r = self.find_best_fit(m, p_ideal, R)
                if r is None:
                    return self.result(False, m)
                R -= r
        return self.result(True, None)

    def _split(self, g, p_ideal):
        self.remain.remove(g)
        t = Gpulet(g.gpu, 0, p_ideal)
        s = Gpulet(g.gpu, 1, 100 - p_ideal)
        self.remain.append(t)
        self.remain.append(s)
        return t, s

    def _unsplit(self, g, t, s):
        self.remain.remove(t)
        self.remain.remove(s)
        self.remain.append(g)

    def find_best_fit(self, m, p_ideal, R):
        # E2 extension (C6 #21b): when no remaining gpu-let is >= p_ideal, the
        # scan is retried with the largest remaining size below p_ideal, then
        # the next smaller one, ... (the literal Alg. 1 would strand them).
        thresholds = [p_ideal] + sorted({g.size for g in self.remain if g.size < p_ideal}, reverse=True)
        for thr in thresholds:
            res = self._scan(m, thr, R)
            if res is not None:
                return res
        return self._merge_only(m, R)

    def _scan(self, m, p_ideal, R):
        chosen, split_info, r = None, None, 0
        for g in sorted(self.remain, key=lambda g: (g.size, g.gpu, g.slot)):
            if g.size < p_ideal:
                continue
            t, si = g, None
            if g.size == 100 and p_ideal < 100 and not self.fixed:
                t, s = self._split(g, p_ideal)                  # Split
                si = (g, t, s)
            A = self.aggregate(self.sibling(t))
            b = self.b_int(m, t.size, A)                        # max b: 2 (L + intf) <= SLO
            ok = b is not None
            if ok:
                F = self.factor(m, b, t.size, A)
                e = self.leff(m, b, t.size, F)
            if ok:
                r = min(R, b * 1_000_000 // e)
                t.lanes = [Lane(m, r)]
                ok = self.sibling_ok(t)
                t.lanes = []
            if not ok:
                if si:
                    self._unsplit(*si)
                continue
            chosen, split_info = t, si
            break
        if chosen is not None:
            for ga in self.alloc:                               # temporal merge
                if any(ln.m == m for ln in ga.lanes):
                    continue
                if self._try_merge(ga, Lane(m, r)):
                    if split_info:                              # RevertSplit
                        self._unsplit(*split_info)
                    return r
            chosen.lanes = [Lane(m, r)]
            self.remain.remove(chosen)
            self.alloc.append(chosen)
            return r
        return None

    def _merge_only(self, m, R):
        # E1 extension (C6 #21): merge-only fallback
        for ga in self.alloc:
            if any(ln.m == m for ln in ga.lanes):
                continue
            c = self.cap(m, ga.size)
            if c <= 0:
                continue
            r = min(R, c)
            if self._try_merge(ga, Lane(m, r)):
                return r
        return None

    def _try_merge(self, ga, lane):
        old = ga.lanes
        ga.lanes = old + [lane]
        if self.feasible(ga) and self.sibling_ok(ga):
            return True
        ga.lanes = old
        return False

    # ---- plan dump (C2.12) ------------------------------------------------------
    def result(self, ok, failed):
        gl = sorted(self.remain + self.alloc, key=lambda g: (g.gpu, g.slot))
        lines = []
        for g in gl:
            d = {"gpu": g.gpu, "slot": g.slot, "size": g.size, "sm": self.P.sm[g.size], "D_us": 0, "lanes": []}
            if g.lanes:
                ev = self.eval_lanes(g, self.aggregate(self.sibling(g)))
                assert ev is not None, "committed lane set became infeasible"
                D, recs = ev
                d["D_us"] = D
                d["lanes"] = [{"model": self.P.names[ln.m], "rate": ln.r, "batch": b,
                               "exec_us": e, "F": F} for ln, b, e, F in recs]
            lines.append(json.dumps(d, separators=(",", ":")))
        lines.append(json.dumps({"verdict": "Schedulable" if ok else "NotSchedulable",
                                 "failed_model": None if failed is None else self.P.names[failed]},
                                separators=(",", ":")))
        return Plan(ok, failed, gl, "\n".join(lines) + "\n")


@dataclass
class Plan:
    ok: bool
    failed: object
    gpulets: list
    dump: str


def knee(rates):
    """C2.4: p_eff from the capacity curve r(p) on GRID, IEEE double, fixed order."""
    rmax = max(rates)
    if rmax == 0:
        return None
    x = [(float(p) - 20.0) / 80.0 for p in GRID]
    y = [float(r) / float(rmax) for r in rates]
    kap = {}
    for i in range(1, len(GRID) - 1):
        h1 = x[i] - x[i - 1]
        h2 = x[i + 1] - x[i]
        s1 = (y[i] - y[i - 1]) / h1
        s2 = (y[i + 1] - y[i]) / h2
        ypp = 2.0 * (s2 - s1) / (h1 + h2)
        yp = (y[i + 1] - y[i - 1]) / (h1 + h2)
        q = 1.0 + yp * yp
        kap[i] = -ypp / (q * math.sqrt(q))
    cands = [i for i in kap if rates[i] > 0 and kap[i] > EPS_KNEE]
    if not cands:
        return 100
    kmax = max(kap[i] for i in cands)
    return min(GRID[i] for i in cands if kap[i] >= kmax - EPS_KNEE)


def curvatures(rates):
    rmax = max(rates)
    x = [(float(p) - 20.0) / 80.0 for p in GRID]
    y = [float(r) / float(rmax) for r in rates]
    out = {}
    for i in range(1, len(GRID) - 1):
        h1, h2 = x[i] - x[i - 1], x[i + 1] - x[i]
        s1, s2 = (y[i] - y[i - 1]) / h1, (y[i + 1] - y[i]) / h2
        ypp = 2.0 * (s2 - s1) / (h1 + h2)
        yp = (y[i + 1] - y[i - 1]) / (h1 + h2)
        q = 1.0 + yp * yp
        out[GRID[i]] = -ypp / (q * math.sqrt(q))
    return out


# ---- C2.9 SBP baseline (whole-GPU temporal sharing) --------------------------------
def sbp(prof, slo, rates, num_gpus, size=100):
    """Squishy bin packing (Nexus), reading C2.9, with every bin a gpu-let
    of `size` %: whole GPUs (100, the temporal-sharing baseline) or both halves of
    evenly split GPUs (50: "SBP algorithm that independently schedules two evenly
    split gpu-lets", Fig. success-case) -> num_gpus * 100 // size bins."""
    S = Scheduler(prof, slo, None, "sbp")
    per = 100 // size
    bins = num_gpus * per
    order = sorted([m for m in range(len(rates)) if rates[m] > 0], key=lambda m: (-rates[m], m))
    gpus = []          # list of lane lists
    residual = []
    failed = None
    for m in order:
        b = S.b_sat(m, size)
        if b is None:
            failed = m
            break
        L = prof.L(m, b, size)
        cap = b * 1_000_000 // L
        k, r = divmod(rates[m], cap)
        for _ in range(k):
            gpus.append([Lane(m, cap)])
        if len(gpus) > bins:
            failed = m
            break
        if r > 0:
            D = L
            bp = (r * D + 999_999) // 1_000_000
            residual.append((m, r, prof.L(m, bp, size), D))
    if failed is None:
        # occupancy e/D descending; exact cross-multiplication; stable in model order
        import functools

        def cmp(a, b):
            lhs, rhs = a[2] * b[3], b[2] * a[3]
            return -1 if lhs > rhs else (1 if lhs < rhs else 0)
        residual.sort(key=functools.cmp_to_key(cmp))
        rgpus = []
        for m, r, _e, _D in residual:
            best, best_occ = None, None
            for gi, lanes in enumerate(rgpus):
                ev = S.eval_lanes(Gpulet(0, 0, size), None, lanes=lanes + [Lane(m, r)])
                if ev is None:
                    continue
                D, recs = ev
                occ = (sum(e for _l, _b, e, _F in recs), D)
                if best is None or occ[0] * best_occ[1] > best_occ[0] * occ[1]:
                    best, best_occ = gi, occ
            if best is None:
                rgpus.append([Lane(m, r)])
            else:
                rgpus[best].append(Lane(m, r))
            if len(gpus) + len(rgpus) > bins:
                failed = m
                break
        gpus += rgpus
    S.remain, S.alloc = [], []
    for i in range(bins):
        g = Gpulet(i // per, i % per, size, list(gpus[i]) if i < len(gpus) else [])
        (S.alloc if g.lanes else S.remain).append(g)
    return S.result(failed is None, failed)


def schedule(prof, slo, rates, num_gpus, mode, coeffs=None):
    """Top-level: mode in {gpulet, gpulet+int, sbp}."""
    if mode == "sbp":
        return sbp(prof, slo, rates, num_gpus)
    if mode == "sbp50":
        return sbp(prof, slo, rates, num_gpus, size=50)
    return Scheduler(prof, slo, coeffs, mode).run(rates, num_gpus)


# ---- C2.10 ideal + brute force -------------------------------------------------------
LAYOUTS = ((100,), (20, 80), (40, 60), (50, 50))


def ideal(prof, slo, rates, num_gpus, mode="gpulet+int", coeffs=None):
    """Exhaustive over multiset layouts, fixed-layout Alg. 1 inside."""
    for combo in combinations_with_replacement(range(len(LAYOUTS)), num_gpus):
        layout = [LAYOUTS[i] for i in combo]
        plan = Scheduler(prof, slo, coeffs, mode).run(rates, num_gpus, layout=layout)
        if plan.ok:
            return plan
    return plan


def brute_force(prof, slo, rates, mode="gpulet+int", coeffs=None):
    """Oracle of the oracle: N = 1, M <= 2, small integer rates.  Enumerates every
    layout, every non-empty gpu-let subset per model and every integer rate split;
    feasible iff every lane set passes C2.6/C2.7.  Returns True/False."""
    S = Scheduler(prof, slo, coeffs, mode)
    models = [m for m in range(len(rates)) if rates[m] > 0]
    for lay in LAYOUTS:
        gls = [Gpulet(0, s, sz) for s, sz in enumerate(lay)]
        subsets = [sub for k in range(1, len(gls) + 1) for sub in _subsets(len(gls), k)]
        for choice in product(subsets, repeat=len(models)):
            for splits in product(*[_compositions(rates[m], len(ch)) for m, ch in zip(models, choice)]):
                for g in gls:
                    g.lanes = []
                for m, ch, sp in zip(models, choice, splits):
                    for gi, r in zip(ch, sp):
                        gls[gi].lanes.append(Lane(m, r))
                S.remain, S.alloc = [], [g for g in gls]
                if all(not g.lanes or S.eval_lanes(g, S.aggregate(S.sibling(g))) is not None for g in gls):
                    return True
    return False


def _subsets(n, k):
    from itertools import combinations
    return list(combinations(range(n), k))


def _compositions(total, parts):
    if parts == 1:
        yield (total,)
        return
    for first in range(1, total - parts + 2):
        for rest in _compositions(total - first, parts - 1):
            yield (first,) + rest
