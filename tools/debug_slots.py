"""Per-slot decode output vs the oracle parse (debug aid)."""
import ctypes
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_07454_b200 as cvlg  # noqa: E402
from oracle.oracle import Ref  # noqa: E402

ref = Ref()
lib = cvlg.cvlg.lib()
lib.cvlg_debug_slots.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
with tempfile.TemporaryDirectory() as d:
    ref.generate_day(d, seed=1, journeys=20, shards=2)
    paths = sorted(str(p) for p in Path(d).glob("*.csv"))
    ctx = cvlg.Context()
    cvlg.run_pipeline(paths, cvlg.GridSpec(), ctx=ctx)
    n = ctypes.c_uint64()
    lib.cvlg_debug_slots(ctx.handle, None, None, None, None, 0, ctypes.byref(n))
    N = n.value
    ts = np.zeros(N, np.int64); sp = np.zeros(N, np.float64); code = np.zeros(N, np.uint32); loff = np.zeros(N, np.uint64)
    lib.cvlg_debug_slots(ctx.handle, ts.ctypes.data_as(ctypes.c_void_p), sp.ctypes.data_as(ctypes.c_void_p),
                         code.ctypes.data_as(ctypes.c_void_p), loff.ctypes.data_as(ctypes.c_void_p), N, ctypes.byref(n))
    blob = b"".join(Path(p).read_bytes() for p in paths)
    cols = [0, 1, 2, 3, 4, 5, 6, 7]
    bad = 0
    for i in range(N):
        e = blob.index(b"\n", int(loff[i]))
        line = blob[int(loff[i]):e]
        why, rec = ref.parse_record(line, cols)
        ok = why == -1 and rec.epoch_sec == ts[i] and rec.speed == sp[i]
        if not ok:
            bad += 1
            if bad < 10:
                print(i, line, why, rec.epoch_sec, ts[i], rec.speed, sp[i], hex(code[i]))
    heads = int((code >> 31).sum())
    print("N", N, "bad", bad, "heads", heads)
