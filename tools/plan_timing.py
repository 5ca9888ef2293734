"""Phase timings of cfg4 searches through the stable search-plan C ABI, for a
given build of the library (A/B and bisection of builds):
    python tools/plan_timing.py lib1.so [lib2.so ...]"""
import ctypes as C
import os
import sys

import numpy as np
import torch


class Cfg(C.Structure):
    _fields_ = [("query_length", C.c_size_t), ("window_ratio", C.c_double),
                ("algorithm", C.c_int32), ("use_lower_bounds", C.c_int32),
                ("tighten_ub", C.c_int32), ("reserved_", C.c_int32)]


def run(path, n=100_000_000, m=1024, ratio=205 / 1024, reps=int(os.environ.get("REPS", "4"))):
    L = C.CDLL(path)
    vp = C.c_void_p
    L.eapdtw_ctx_create.argtypes = [C.POINTER(vp), C.c_int]
    L.eapdtw_random_walk_normal.argtypes = [C.c_size_t, C.c_uint64, C.POINTER(C.c_double)]
    L.eapdtw_search_plan_create.argtypes = [vp, vp, C.c_size_t, C.POINTER(C.c_double), C.c_size_t,
                                            C.POINTER(Cfg), C.c_uint64, C.POINTER(vp)]
    for f in ("eapdtw_search_plan_prepare", "eapdtw_search_plan_reset", "eapdtw_search_plan_destroy"):
        getattr(L, f).argtypes = [vp]
    L.eapdtw_search_plan_run.argtypes = [vp, C.c_size_t, C.c_size_t]
    L.eapdtw_search_plan_timings.argtypes = [vp, C.POINTER(C.c_float)]
    L.eapdtw_search_plan_result.argtypes = [vp, C.c_char_p]
    ctx = vp()
    assert L.eapdtw_ctx_create(C.byref(ctx), 0) == 0
    for kv in filter(None, os.environ.get("OPTS", "").split(",")):
        k, v = kv.split("=")
        L.eapdtw_ctx_set_option.argtypes = [vp, C.c_char_p, C.c_longlong]
        assert L.eapdtw_ctx_set_option(ctx, k.encode(), int(v)) == 0, kv
    ref = np.empty(n)
    q = np.empty(m)
    L.eapdtw_random_walk_normal(n, 20261019, ref.ctypes.data_as(C.POINTER(C.c_double)))
    L.eapdtw_random_walk_normal(m, 20261020, q.ctypes.data_as(C.POINTER(C.c_double)))
    dref = torch.from_numpy(ref).cuda()
    cfg = Cfg(0, ratio, 2, 1, 1, 0)
    plan = vp()
    assert L.eapdtw_search_plan_create(ctx, vp(dref.data_ptr()), n, q.ctypes.data_as(C.POINTER(C.c_double)),
                                       m, C.byref(cfg), 0, C.byref(plan)) == 0
    rows = []
    for k in range(reps):
        L.eapdtw_search_plan_reset(plan)
        assert L.eapdtw_search_plan_prepare(plan) == 0
        assert L.eapdtw_search_plan_run(plan, 0, n - m + 1) == 0
        t = (C.c_float * 4)()
        assert L.eapdtw_search_plan_timings(plan, t) == 0
        buf = C.create_string_buffer(256)
        L.eapdtw_search_plan_result(plan, buf)
        rows.append(list(t))
    L.eapdtw_search_plan_destroy(plan)
    med = np.median(np.array(rows[1:]), axis=0)
    print(f"{path} {os.environ.get('OPTS', '')}: stats {med[0]:.3f} env {med[1]:.3f} warm {med[2]:.3f} sweep {med[3]:.3f} total {med.sum():.3f}",
          flush=True)


if __name__ == "__main__":
    # CFG=cfg2|cfg3|cfg4 (bench.py's sizes)
    size = {"cfg2": (1_000_000, 128, 0.05), "cfg3": (10_000_000, 512, 0.1),
            "cfg4": (100_000_000, 1024, 205 / 1024)}[os.environ.get("CFG", "cfg4")]
    for p in sys.argv[1:]:
        run(p, *size)
