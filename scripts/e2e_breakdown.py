"""Host-side phases of one end-to-end batch (config 5): validate+upload, run, fetch."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import capi, synth  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
ds = synth.make(5, scale)
s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
pool = xb.DevicePool(s, ds.symbols, ds.offsets)
L = capi.lib()
t = xb.xband.tasks_array(ds.tasks)
out = np.zeros(2 * len(t), dtype=capi.RESULT_DTYPE)
ss = np.zeros(len(t), dtype=np.int32)
ex = capi.make_exec(1, [0], None, 0)
for rep in range(3):
    pool.evict()
    err, bad = C.c_int(0), C.c_int64(-1)
    t0 = time.perf_counter()
    b = L.xb_batch_create(pool._h, t.ctypes.data, len(t), ds.k, ds.band, C.byref(ex), C.byref(bad), C.byref(err))
    t1 = time.perf_counter()
    capi.check(L.xb_batch_run(b), "run")
    t2 = time.perf_counter()
    capi.check(L.xb_batch_sync(b), "sync")
    t3 = time.perf_counter()
    capi.check(L.xb_batch_fetch(b, out.ctypes.data, ss.ctypes.data), "fetch")
    t4 = time.perf_counter()
    st = capi.XbStats()
    L.xb_batch_stats(b, C.byref(st))
    L.xb_batch_free(b)
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms  run-launch {1e3*(t2-t1):.1f}  sync {1e3*(t3-t2):.1f}  "
          f"fetch {1e3*(t4-t3):.1f}  free {1e3*(t5-t4):.1f}  total {1e3*(t5-t0):.1f}  device {st.ms_total:.1f}  "
          f"h2d {st.h2d_bytes/1e6:.0f} MB", flush=True)

# the batch stream (bench e2e): host phases of each batch, one batch in flight ahead
pools = [pool, xb.DevicePool(s, ds.symbols, ds.offsets)]
for n_batches in (2, 6):
    t0 = time.perf_counter()
    ms = lambda: 1e3 * (time.perf_counter() - t0)  # noqa: E731
    prev, log = None, []
    for i in range(n_batches + 1):
        if i < n_batches:
            pools[i % 2].evict()
            err, bad = C.c_int(0), C.c_int64(-1)
            a = ms()
            h = L.xb_batch_create(pools[i % 2]._h, t.ctypes.data, len(t), ds.k, ds.band, C.byref(ex),
                                  C.byref(bad), C.byref(err))
            b = ms()
            capi.check(L.xb_batch_run(h), "run")
            c = ms()
            log.append(f"b{i}: create {a:.0f}-{b:.0f} run -{c:.0f}")
        if prev is not None:
            a = ms()
            capi.check(L.xb_batch_fetch(prev, out.ctypes.data, ss.ctypes.data), "fetch")
            st = capi.XbStats()
            L.xb_batch_stats(prev, C.byref(st))
            L.xb_batch_free(prev)
            log.append(f"fetch b{i-1} {a:.0f}-{ms():.0f} (device {st.ms_total:.1f})")
        prev = h if i < n_batches else None
    print(f"stream of {n_batches}: wall {ms():.0f} ms: " + "; ".join(log), flush=True)
