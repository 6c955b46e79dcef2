"""Thin ctypes binding of include/gpulet.h (argument marshalling only).

Every step of the hot path runs inside libgpulet.so (CUDA kernels + native
runtime + native scheduler).  There is no fallback: if the library or a GPU is
missing, calls raise GpuletError.  torch is used only to hand over device
pointers of tensors the caller allocated.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgpulet.so")

GL_OK = 0
ERRORS = {-1: "GL_E_ARG", -2: "GL_E_GRID", -3: "GL_E_CAPACITY", -4: "GL_E_PARTITION", -5: "GL_E_STATE",
          -6: "GL_E_MODEL", -7: "GL_E_QUEUE_FULL", -8: "GL_E_NOT_CONCURRENT", -9: "GL_E_PARSE",
          -10: "GL_E_DATA", -11: "GL_E_BUDGET", -12: "GL_E_CUDA", -13: "GL_E_TIMEOUT"}
MODELS = ["lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base"]
MODES = {"gpulet": 0, "gpulet+int": 1, "sbp": 2, "ideal": 3, "sbp50": 4}

# exported symbols declared in include/gpulet.h
SYMBOLS = ["gl_init", "gl_shutdown", "gl_last_error", "gl_load_model", "gl_model_io", "gl_model_cost",
           "gl_create_gpulet", "gl_create_gpulets", "gl_create_gpulets_unconfined", "gl_destroy_gpulet", "gl_gpulet_smids", "gl_submit_batch", "gl_poll", "gl_wait",
           "gl_profile", "gl_profile_tail", "gl_run_once", "gl_program_info", "gl_serve", "gl_serve_sim", "gl_serve_chain", "gl_serve_sim_chain", "gl_schedule", "gl_profile_load",
           "gl_workload_rates", "gl_schedule_files", "gl_bw_probe", "gl_publish_probe", "gl_floor", "gl_fit_interference", "gl_test_gemm", "gl_test_conv", "gl_test_misc",
           "gl_test_stats", "gl_set_tuning", "gl_ssd_detect_workspace", "gl_ssd_detect", "gl_crop_resize"]


class GpuletError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Completion(ctypes.Structure):
    _fields_ = [("ticket", ctypes.c_uint64), ("gpulet", ctypes.c_int32), ("model", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("status", ctypes.c_int32), ("t_submit_ns", ctypes.c_uint64),
                ("t_dequeue_ns", ctypes.c_uint64), ("t_start_ns", ctypes.c_uint64), ("t_end_ns", ctypes.c_uint64)]


class SchedInput(ctypes.Structure):
    _fields_ = [("n_models", ctypes.c_int32), ("names", ctypes.POINTER(ctypes.c_char_p)),
                ("lat_us", ctypes.POINTER(ctypes.c_int32)), ("l2", ctypes.POINTER(ctypes.c_double)),
                ("mem", ctypes.POINTER(ctypes.c_double)), ("slo_us", ctypes.POINTER(ctypes.c_int32)),
                ("rates", ctypes.POINTER(ctypes.c_int32)), ("coeffs", ctypes.c_double * 5),
                ("num_gpus", ctypes.c_int32), ("mode", ctypes.c_int32), ("sm_count", ctypes.POINTER(ctypes.c_int32))]


class Lane(ctypes.Structure):
    _fields_ = [("gpulet", ctypes.c_int32), ("model_id", ctypes.c_int32), ("model_slot", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("duty_us", ctypes.c_int32), ("weight", ctypes.c_int32),
                ("drop_us", ctypes.c_int32), ("margin_us", ctypes.c_int32), ("in_dev", ctypes.c_void_p),
                ("out_dev", ctypes.c_void_p), ("in_host", ctypes.c_void_p), ("out_host", ctypes.c_void_p),
                ("in_req_bytes", ctypes.c_int64), ("out_req_bytes", ctypes.c_int64), ("host_slots", ctypes.c_int32),
                ("pad2_", ctypes.c_int32), ("in_dev2", ctypes.c_void_p), ("out_dev2", ctypes.c_void_p),
                ("leff_us", ctypes.POINTER(ctypes.c_int32))]


class Chain(ctypes.Structure):
    """gl_chain (include/gpulet.h): two-stage application chains (F3)."""
    _fields_ = [("spawn", ctypes.POINTER(ctypes.c_int32)), ("handoff_us", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("cap_req", ctypes.c_int64), ("parent", ctypes.POINTER(ctypes.c_int32)),
                ("req_model", ctypes.POINTER(ctypes.c_int32)), ("n_total", ctypes.c_int64)]


_lib = None


def lib():
    """Load libgpulet.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        path = os.environ.get("GL_LIB", LIB_PATH)   # GL_LIB: an alternative in-tree build (A/B tuning runs)
        if not os.path.exists(path):
            raise GpuletError(-12, f"{path} missing: run `python -m paper_2109_01611_b200.build`")
        L = ctypes.CDLL(path)
        P, I32, I64, U64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        sig = {
            "gl_init": [ctypes.c_int, ctypes.POINTER(P)],
            "gl_shutdown": [P],
            "gl_load_model": [P, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(I32)],
            "gl_model_io": [P, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)],
            "gl_model_cost": [P, I32, I32, ctypes.POINTER(D), ctypes.POINTER(D)],
            "gl_create_gpulet": [P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(I32), ctypes.POINTER(I32)],
            "gl_create_gpulets": [P, ctypes.c_int, I32, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32)],
            "gl_create_gpulets_unconfined": [P, ctypes.c_int, I32, ctypes.POINTER(I32), ctypes.POINTER(I32),
                                             ctypes.POINTER(I32)],
            "gl_destroy_gpulet": [P, I32],
            "gl_gpulet_smids": [P, I32, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)],
            "gl_submit_batch": [P, I32, I32, P, P, I32, ctypes.c_float, ctypes.POINTER(U64)],
            "gl_poll": [P, ctypes.POINTER(Completion), I32, ctypes.POINTER(I32)],
            "gl_wait": [P, U64, I32, ctypes.POINTER(Completion)],
            "gl_profile": [P, I32, I32, I32, I32, I32, P, P, ctypes.POINTER(D)],
            "gl_profile_tail": [P, I32, I32, I32, I32, I32, P, P, D, ctypes.POINTER(D), ctypes.POINTER(D)],
            "gl_run_once": [P, I32, I32, P, P, I32, ctypes.POINTER(U64), I32, ctypes.POINTER(I32)],
            "gl_program_info": [P, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(D),
                                ctypes.POINTER(D), I32, ctypes.POINTER(I32)],
            "gl_serve": [P, ctypes.POINTER(Lane), I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I32), I64,
                         ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(U64), ctypes.POINTER(I64),
                         ctypes.POINTER(I64), ctypes.POINTER(ctypes.c_int64)],
            "gl_serve_sim": [ctypes.POINTER(Lane), I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I32), I64,
                             ctypes.POINTER(I32), ctypes.POINTER(I64), ctypes.POINTER(I64), I64, ctypes.POINTER(I64)],
            "gl_serve_chain": [P, ctypes.POINTER(Lane), I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I32), I64,
                               ctypes.POINTER(I32), ctypes.POINTER(Chain), ctypes.POINTER(I64), ctypes.POINTER(U64),
                               ctypes.POINTER(ctypes.c_int64)],
            "gl_serve_sim_chain": [ctypes.POINTER(Lane), I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I32), I64,
                                   ctypes.POINTER(I32), ctypes.POINTER(Chain), ctypes.POINTER(I64), ctypes.POINTER(I64),
                                   I64, ctypes.POINTER(I64)],
            "gl_schedule": [ctypes.POINTER(SchedInput), ctypes.c_char_p, ctypes.c_size_t,
                            ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(I32)],
            "gl_profile_load": [ctypes.c_char_p, I32, ctypes.POINTER(I32), ctypes.POINTER(D), ctypes.POINTER(D),
                                ctypes.POINTER(I32)],
            "gl_workload_rates": [ctypes.POINTER(I32), I32, ctypes.c_char_p, D, I32, ctypes.POINTER(I32),
                                  ctypes.POINTER(I32)],
            "gl_schedule_files": [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t,
                                  ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(I32)],
            "gl_fit_interference": [ctypes.POINTER(D), ctypes.POINTER(D), I32, ctypes.POINTER(D)],
            "gl_publish_probe": [P, ctypes.c_int, I32, ctypes.POINTER(D), ctypes.POINTER(D)],
            "gl_floor": [P, I32, I32, I32, ctypes.POINTER(D), ctypes.POINTER(D)],
            "gl_bw_probe": [P, ctypes.c_int, ctypes.c_int, I64, I32, ctypes.POINTER(D), ctypes.POINTER(I32)],
            "gl_test_gemm": [P, ctypes.c_int, P, P, P, P, I32, I32, I32, I32, I32, I32, I32, I32],
            "gl_test_conv": [P, ctypes.c_int, P, P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, I32, I32],
            "gl_test_misc": [P, ctypes.c_int, I32, ctypes.POINTER(I32), I32, P, I64, P, P],
            "gl_test_stats": [ctypes.POINTER(U64), ctypes.POINTER(U64), I32, ctypes.POINTER(I32)],
            "gl_set_tuning": [I32, I32],
            "gl_ssd_detect_workspace": [I32, I32, ctypes.POINTER(ctypes.c_size_t)],
            "gl_ssd_detect": [P, P, I32, ctypes.c_float, ctypes.c_float, I32, I32, P, P, P, ctypes.c_size_t, P],
            "gl_crop_resize": [P, I32, I32, I32, I32, P, P, I32, I32, I32, I32, P, P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = I32
        L.gl_last_error.restype = ctypes.c_char_p
        L.gl_last_error.argtypes = []
        _lib = L
    return _lib


def _check(rc):
    if rc != GL_OK:
        raise GpuletError(rc, lib().gl_last_error().decode(errors="replace"))


def _ptr(x):
    """Device/host address of a torch tensor, numpy array or int (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(type(x))


def _lanes(lanes):
    """gl_lane array from lane dicts (routing / dispatch fields; leff_us: 32 ints or absent)."""
    import numpy as np
    L = (Lane * len(lanes))()
    keep = []
    for i, d in enumerate(lanes):
        L[i].gpulet, L[i].model_id, L[i].model_slot = d["gpulet"], d.get("model_id", 0), d["model_slot"]
        L[i].batch, L[i].duty_us, L[i].weight, L[i].drop_us = d["batch"], d["duty_us"], d["weight"], d["drop_us"]
        L[i].margin_us = d.get("margin_us", 0)
        if d.get("leff_us") is not None:
            a = np.ascontiguousarray(d["leff_us"], dtype=np.int32)
            assert a.size == 32
            keep.append(a)
            L[i].leff_us = a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    return L, keep


def serve_sim(lanes, n_models, arr_us, arr_model, slo_us, cap=1 << 20):
    """gl_serve_sim (virtual clock, no GPU) -> (lat_us int64 ndarray, batch log [(lane, t, k, first)])."""
    import numpy as np
    L, keep = _lanes(lanes)
    a = np.ascontiguousarray(arr_us, dtype=np.int64)
    m = np.ascontiguousarray(arr_model, dtype=np.int32)
    s = np.ascontiguousarray(slo_us, dtype=np.int32)
    lat = np.zeros(len(a), np.int64)
    log = np.zeros((cap, 4), np.int64)
    n = ctypes.c_int64()
    P64 = ctypes.POINTER(ctypes.c_int64)
    _check(lib().gl_serve_sim(L, len(lanes), n_models, a.ctypes.data_as(P64),
                              m.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(a),
                              s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), lat.ctypes.data_as(P64),
                              log.ctypes.data_as(P64), cap, ctypes.byref(n)))
    assert n.value <= cap
    return lat, [tuple(int(v) for v in row) for row in log[:n.value]]


def _chain(n_models, spawn, handoff_us, n_req):
    """spawn: {model slot: [spawned model slots]} -> (gl_chain, buffers kept alive, cap)."""
    import numpy as np
    sp = np.zeros((n_models, n_models), np.int32)
    for m, kids in spawn.items():
        for k in kids:
            sp[m, k] += 1
    fan = max(1, int(sp.sum(1).max()) + 1)
    cap = n_req * fan          # a chain of depth 1 (trace -> spawned); deeper chains: pass a larger cap
    par = np.zeros(cap, np.int32)
    mdl = np.zeros(cap, np.int32)
    P32 = ctypes.POINTER(ctypes.c_int32)
    c = Chain(sp.ctypes.data_as(P32), int(handoff_us), 0, cap, par.ctypes.data_as(P32), mdl.ctypes.data_as(P32), 0)
    return c, (sp, par, mdl), cap


def serve_sim_chain(lanes, n_models, arr_us, arr_model, slo_us, spawn, handoff_us, cap=1 << 20):
    """gl_serve_sim_chain -> (lat_us, batch log, parent, model) over trace + spawned requests."""
    import numpy as np
    L, keep = _lanes(lanes)
    a = np.ascontiguousarray(arr_us, dtype=np.int64)
    m = np.ascontiguousarray(arr_model, dtype=np.int32)
    s = np.ascontiguousarray(slo_us, dtype=np.int32)
    ch, bufs, creq = _chain(n_models, spawn, handoff_us, len(a))
    lat = np.zeros(creq, np.int64)
    log = np.zeros((cap, 4), np.int64)
    n = ctypes.c_int64()
    P64 = ctypes.POINTER(ctypes.c_int64)
    _check(lib().gl_serve_sim_chain(L, len(lanes), n_models, a.ctypes.data_as(P64),
                                    m.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(a),
                                    s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(ch),
                                    lat.ctypes.data_as(P64), log.ctypes.data_as(P64), cap, ctypes.byref(n)))
    t = ch.n_total
    return lat[:t], [tuple(int(v) for v in row) for row in log[:n.value]], bufs[1][:t].copy(), bufs[2][:t].copy()


class Context:
    """gl_ctx wrapper: models, gpu-lets, submit/poll."""

    def __init__(self, num_gpus=1):
        self.h = ctypes.c_void_p()
        _check(lib().gl_init(num_gpus, ctypes.byref(self.h)))

    def close(self):
        if self.h:
            lib().gl_shutdown(self.h)
            self.h = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def load_model(self, gpu, kind, weight_file):
        k = MODELS.index(kind) if isinstance(kind, str) else kind
        mid = ctypes.c_int32()
        _check(lib().gl_load_model(self.h, gpu, k, weight_file.encode(), ctypes.byref(mid)))
        return mid.value

    def model_io(self, mid, batch):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().gl_model_io(self.h, mid, batch, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def model_cost(self, mid, batch):
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(lib().gl_model_cost(self.h, mid, batch, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def create_gpulet(self, gpu, sm_pct):
        gid, n = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().gl_create_gpulet(self.h, gpu, sm_pct, ctypes.byref(gid), ctypes.byref(n)))
        return gid.value, n.value

    def create_gpulets(self, gpu, pcts, unconfined=False):
        """Partition a GPU into len(pcts) gpu-lets at once; returns [(id, sm_count)].
        unconfined: the F4 "MPS(default)" analogue (gl_create_gpulets_unconfined)."""
        n = len(pcts)
        p = (ctypes.c_int32 * n)(*pcts)
        ids = (ctypes.c_int32 * n)()
        sms = (ctypes.c_int32 * n)()
        fn = lib().gl_create_gpulets_unconfined if unconfined else lib().gl_create_gpulets
        _check(fn(self.h, gpu, n, p, ids, sms))
        return [(ids[i], sms[i]) for i in range(n)]

    def destroy_gpulet(self, gid):
        _check(lib().gl_destroy_gpulet(self.h, gid))

    def gpulet_smids(self, gid, cap=160):
        buf = (ctypes.c_int32 * cap)()
        n = ctypes.c_int32()
        _check(lib().gl_gpulet_smids(self.h, gid, buf, cap, ctypes.byref(n)))
        return list(buf[: n.value])

    def submit_batch(self, gid, mid, x, y, batch, slo_ms=0.0):
        t = ctypes.c_uint64()
        _check(lib().gl_submit_batch(self.h, gid, mid, _ptr(x), _ptr(y), batch, slo_ms, ctypes.byref(t)))
        return t.value

    def try_submit_batch(self, gid, mid, x, y, batch, slo_ms=0.0):
        """Like submit_batch but returns None when the ring is full."""
        t = ctypes.c_uint64()
        rc = lib().gl_submit_batch(self.h, gid, mid, _ptr(x), _ptr(y), batch, slo_ms, ctypes.byref(t))
        if rc == -7:
            return None
        _check(rc)
        return t.value

    def poll(self, max_n=256):
        buf = (Completion * max_n)()
        n = ctypes.c_int32()
        _check(lib().gl_poll(self.h, buf, max_n, ctypes.byref(n)))
        return [buf[i] for i in range(n.value)]

    def wait(self, ticket, timeout_ms=60000):
        c = Completion()
        _check(lib().gl_wait(self.h, ticket, timeout_ms, ctypes.byref(c)))
        return c

    def profile(self, gid, mid, batch, x, y, warmup=10, reps=50):
        d = ctypes.c_double()
        _check(lib().gl_profile(self.h, gid, mid, batch, warmup, reps, _ptr(x), _ptr(y), ctypes.byref(d)))
        return d.value

    def profile_tail(self, gid, mid, batch, x, y, warmup=10, reps=200, q=0.99):
        """gl_profile_tail -> (median, q-quantile) µs host-observed service latency."""
        d, t = ctypes.c_double(), ctypes.c_double()
        _check(lib().gl_profile_tail(self.h, gid, mid, batch, warmup, reps, _ptr(x), _ptr(y), float(q),
                                     ctypes.byref(d), ctypes.byref(t)))
        return d.value, t.value

    def run_once(self, mid, batch, x, y, n_sm=0, trace=True, roles=False):
        """One-shot executor launch; returns per-step durations (ns) when trace
        (and, with roles, CTA 0's per-step role stamps relative to step start:
        producer start/end, MMA first/last, epilogue first/end, barrier in/out)."""
        cap = 1024 + 8 * 1000 if roles else 1024
        tr = (ctypes.c_uint64 * cap)()
        n = ctypes.c_int32()
        _check(lib().gl_run_once(self.h, mid, batch, _ptr(x), _ptr(y), n_sm, tr if trace else None, cap,
                                 ctypes.byref(n)))
        if not trace:
            return None
        ts = list(tr[: n.value + 1])
        durs = [ts[i + 1] - ts[i] for i in range(n.value)]
        if not roles:
            return durs
        rl = []
        for s in range(n.value):
            st = list(tr[1024 + 8 * s: 1024 + 8 * s + 8])
            rl.append([(v - ts[s]) if v else None for v in st])
        return durs, rl

    def serve(self, lanes, n_models, arr_us, arr_model, slo_us, stats=False):
        """gl_serve: lanes = list of dicts (gpulet, model_id, model_slot, batch, duty_us,
        weight, drop_us, x, y[, x_host, y_host, in_req_bytes, out_req_bytes, host_slots[, x2, y2]]);
        returns per-request latency (us, -1 dropped), and with stats also
        {"dev_ns": (first dequeue, last end), "h2d_bytes", "d2h_bytes"}."""
        import numpy as np
        L, keep = _lanes(lanes)
        for i, d in enumerate(lanes):
            L[i].in_dev, L[i].out_dev = _ptr(d["x"]), _ptr(d["y"])
            if d.get("x_host") is not None:
                L[i].in_host, L[i].out_host = _ptr(d["x_host"]), _ptr(d["y_host"])
                L[i].in_req_bytes, L[i].out_req_bytes = d["in_req_bytes"], d["out_req_bytes"]
                L[i].host_slots = d["host_slots"]
                if d.get("x2") is not None:
                    L[i].in_dev2, L[i].out_dev2 = _ptr(d["x2"]), _ptr(d["y2"])
        a = np.ascontiguousarray(arr_us, dtype=np.int64)
        m = np.ascontiguousarray(arr_model, dtype=np.int32)
        s = np.ascontiguousarray(slo_us, dtype=np.int32)
        out = np.zeros(len(a), dtype=np.int64)
        dev = (ctypes.c_uint64 * 2)()
        hb, db = ctypes.c_int64(), ctypes.c_int64()
        ls = (ctypes.c_int64 * (4 * len(lanes)))()   # gl_lane_stats[n_lanes]
        _check(lib().gl_serve(self.h, L, len(lanes), n_models, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              m.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(a),
                              s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), dev, ctypes.byref(hb),
                              ctypes.byref(db), ls))
        if stats:
            lanes_st = [{"batches": ls[4 * i], "requests": ls[4 * i + 1], "busy_ns": ls[4 * i + 2] & (2**64 - 1)}
                        for i in range(len(lanes))]
            return out, {"dev_ns": (dev[0], dev[1]), "h2d_bytes": hb.value, "d2h_bytes": db.value,
                         "lanes": lanes_st}
        return out

    def serve_chain(self, lanes, n_models, arr_us, arr_model, slo_us, spawn, handoff_us, stats=False):
        """gl_serve_chain (device-resident lanes): returns (lat_us, parent, model) over the
        trace + spawned requests, and with stats {"dev_ns", "lanes"}."""
        import numpy as np
        L, keep = _lanes(lanes)
        for i, d in enumerate(lanes):
            L[i].in_dev, L[i].out_dev = _ptr(d["x"]), _ptr(d["y"])
        a = np.ascontiguousarray(arr_us, dtype=np.int64)
        m = np.ascontiguousarray(arr_model, dtype=np.int32)
        s = np.ascontiguousarray(slo_us, dtype=np.int32)
        ch, bufs, creq = _chain(n_models, spawn, handoff_us, len(a))
        out = np.zeros(creq, dtype=np.int64)
        dev = (ctypes.c_uint64 * 2)()
        ls = (ctypes.c_int64 * (4 * len(lanes)))()
        _check(lib().gl_serve_chain(self.h, L, len(lanes), n_models, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    m.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), len(a),
                                    s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.byref(ch),
                                    out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), dev, ls))
        t = ch.n_total
        res = (out[:t], bufs[1][:t].copy(), bufs[2][:t].copy())
        if stats:
            lanes_st = [{"batches": ls[4 * i], "requests": ls[4 * i + 1], "busy_ns": ls[4 * i + 2] & (2**64 - 1)}
                        for i in range(len(lanes))]
            return res + ({"dev_ns": (dev[0], dev[1]), "lanes": lanes_st},)
        return res

    def floor(self, gid, warmup=10, reps=200):
        """gl_floor -> (median host round trip µs, median device start -> end µs) of an empty program."""
        h, d = ctypes.c_double(), ctypes.c_double()
        _check(lib().gl_floor(self.h, gid, warmup, reps, ctypes.byref(h), ctypes.byref(d)))
        return h.value, d.value

    def publish_probe(self, gpu=0, reps=1000):
        """gl_publish_probe -> (median, p99) µs of a 64-B descriptor H2D copy + completion."""
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(lib().gl_publish_probe(self.h, gpu, reps, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def bw_probe(self, gpu, sm_pct, nbytes=1 << 30, reps=10):
        """gl_bw_probe -> (GB/s read + write, SMs)."""
        g, n = ctypes.c_double(), ctypes.c_int32()
        _check(lib().gl_bw_probe(self.h, gpu, sm_pct, int(nbytes), reps, ctypes.byref(g), ctypes.byref(n)))
        return g.value, n.value

    def program_info(self, mid, batch, cap=1024):
        t = (ctypes.c_int32 * cap)()
        o = (ctypes.c_int32 * cap)()
        f = (ctypes.c_double * cap)()
        b = (ctypes.c_double * cap)()
        n = ctypes.c_int32()
        _check(lib().gl_program_info(self.h, mid, batch, t, o, f, b, cap, ctypes.byref(n)))
        return [(t[i], o[i], f[i], b[i]) for i in range(n.value)]

    # ---- kernel unit entry points -------------------------------------------
    def test_gemm(self, gpu, A, W_bits, b_bits, out, M, N, K, act=0, swap_ab=0, splitk=1, out_fp32=0, in_ws=0):
        _check(lib().gl_test_gemm(self.h, gpu, _ptr(A), _ptr(W_bits), _ptr(b_bits), _ptr(out), M, N, K, act,
                                  swap_ab, splitk, out_fp32, in_ws))

    def test_conv(self, gpu, x, W_bits, b_bits, y, N, H, W, C, Cout, KH, stride, pad, act=1, in_ws=0):
        _check(lib().gl_test_conv(self.h, gpu, _ptr(x), _ptr(W_bits), _ptr(b_bits), _ptr(y), N, H, W, C, Cout, KH,
                                  stride, pad, act, in_ws))

    @staticmethod
    def test_stats(n_cta=148):
        """(device ns of the last test run, timeline[n_cta][tiles][4] ns or 0)."""
        import numpy as np
        ns = ctypes.c_uint64()
        per = ctypes.c_int32()
        _check(lib().gl_test_stats(ctypes.byref(ns), None, 0, ctypes.byref(per)))
        tl = np.zeros(n_cta * per.value, dtype=np.uint64)
        _check(lib().gl_test_stats(None, tl.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), tl.size, None))
        return ns.value, tl.reshape(n_cta, per.value // 4, 4)

    @staticmethod
    def set_tuning(key, value):
        _check(lib().gl_set_tuning(int(key), int(value)))

    def test_misc(self, gpu, op, iargs, params, x, y):
        ia = (ctypes.c_int32 * len(iargs))(*iargs)
        n = 0 if params is None else int(params.size)
        _check(lib().gl_test_misc(self.h, gpu, op, ia, len(iargs), _ptr(params), n, _ptr(x), _ptr(y)))


def ssd_detect_workspace(n_img, top_k):
    n = ctypes.c_size_t()
    _check(lib().gl_ssd_detect_workspace(int(n_img), int(top_k), ctypes.byref(n)))
    return n.value


def ssd_detect(loc, conf, n_img, det, count, ws, score_thr=0.05, iou_thr=0.45, top_k=200, max_det=100, stream=0):
    """gl_ssd_detect (F3, R27) on device tensors; asynchronous on `stream`."""
    _check(lib().gl_ssd_detect(_ptr(loc), _ptr(conf), int(n_img), float(score_thr), float(iou_thr), int(top_k),
                               int(max_det), _ptr(det), _ptr(count), _ptr(ws), int(ws.numel() * ws.element_size()),
                               stream or None))


def crop_resize(img, n_img, H, W, det, count, max_det, per_img, out, OH=224, OW=224, C=8, stream=0):
    """gl_crop_resize (F3, R27) on device tensors; asynchronous on `stream`."""
    _check(lib().gl_crop_resize(_ptr(img), int(n_img), int(H), int(W), int(C), _ptr(det), _ptr(count), int(max_det),
                                int(per_img), int(OH), int(OW), _ptr(out), stream or None))


def schedule(names, lat_us, l2, mem, slo_us, rates, num_gpus, mode, coeffs=(0, 0, 0, 0, 0), cap=1 << 20,
             sm_count=None):
    """gl_schedule: returns (plan_dump_text, schedulable).  lat_us [M][32][6] ints,
    l2/mem [M][6][6] floats (or None), slo_us/rates [M] ints, sm_count [6] or None."""
    import numpy as np
    M = len(names)
    nm = (ctypes.c_char_p * M)(*[n.encode() for n in names])
    lat = np.ascontiguousarray(lat_us, dtype=np.int32).reshape(-1)
    l2a = np.ascontiguousarray(l2 if l2 is not None else np.zeros((M, 6, 6)), dtype=np.float64).reshape(-1)
    mema = np.ascontiguousarray(mem if mem is not None else np.zeros((M, 6, 6)), dtype=np.float64).reshape(-1)
    slo = np.ascontiguousarray(slo_us, dtype=np.int32)
    rt = np.ascontiguousarray(rates, dtype=np.int32)
    si = SchedInput()
    si.n_models = M
    si.names = nm
    si.lat_us = lat.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    si.l2 = l2a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    si.mem = mema.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    si.slo_us = slo.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    si.rates = rt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    for i in range(5):
        si.coeffs[i] = float(coeffs[i]) if coeffs is not None else 0.0
    si.num_gpus = num_gpus
    si.mode = MODES[mode] if isinstance(mode, str) else mode
    if sm_count is not None:
        sma = np.ascontiguousarray(sm_count, dtype=np.int32)
        si.sm_count = sma.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    buf = ctypes.create_string_buffer(cap)
    ln, verdict = ctypes.c_size_t(), ctypes.c_int32()
    _check(lib().gl_schedule(ctypes.byref(si), buf, cap, ctypes.byref(ln), ctypes.byref(verdict)))
    return buf.value.decode(), bool(verdict.value)


def profile_load(path, strict=False):
    """gl_profile_load -> (lat_us [6][32][6] int32 ndarray, l2 [6][6][6], mem [6][6][6], sm_count [6])."""
    import numpy as np
    lat = np.zeros((6, 32, 6), np.int32)
    l2 = np.zeros((6, 6, 6), np.float64)
    mem = np.zeros((6, 6, 6), np.float64)
    sm = np.zeros(6, np.int32)
    _check(lib().gl_profile_load(os.fsencode(path), 1 if strict else 0,
                                 lat.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                 l2.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 mem.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 sm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return lat, l2, mem, sm


def workload_rates(lat_us, scenario, x=1.0, num_gpus=1, slo_mode="rule"):
    """gl_workload_rates -> (slo_us [6], rates [6]) as Python int lists."""
    import numpy as np
    lat = np.ascontiguousarray(lat_us, dtype=np.int32)
    slo = np.zeros(6, np.int32)
    rates = np.zeros(6, np.int32)
    _check(lib().gl_workload_rates(lat.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   {"rule": 0, "table": 1}[slo_mode], scenario.encode(), float(x), num_gpus,
                                   slo.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   rates.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
    return [int(v) for v in slo], [int(v) for v in rates]


def schedule_files(profile_csv, coeffs_json, workload_json, cap=1 << 20):
    """gl_schedule_files: paths (or inline JSON text for coeffs / workload; dicts are
    serialised) -> (header dict, plan dump text without the header, schedulable)."""
    import json
    if isinstance(workload_json, dict):
        workload_json = json.dumps(workload_json)
    if isinstance(coeffs_json, dict):
        coeffs_json = json.dumps(coeffs_json)
    buf = ctypes.create_string_buffer(cap)
    ln, verdict = ctypes.c_size_t(), ctypes.c_int32()
    _check(lib().gl_schedule_files(os.fsencode(profile_csv),
                                   None if coeffs_json is None else os.fsencode(coeffs_json),
                                   os.fsencode(workload_json), buf, cap, ctypes.byref(ln), ctypes.byref(verdict)))
    text = buf.value.decode()
    head, _, dump = text.partition("\n")
    return json.loads(head), dump, bool(verdict.value), text


def fit_interference(X, y):
    """gl_fit_interference: OLS coefficients c1..c5."""
    import numpy as np
    Xa = np.ascontiguousarray(X, dtype=np.float64)
    ya = np.ascontiguousarray(y, dtype=np.float64)
    c = np.zeros(5)
    _check(lib().gl_fit_interference(Xa.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     ya.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(ya),
                                     c.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return c
