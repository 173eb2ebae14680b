"""R(128) vs buffer size for cudaMalloc / VMM / pool (TLB reach)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1801_05857_b200._lib import check, lib  # noqa: E402

for kind in (0, 1, 2):
    for gb in (48, 96, 144):
        ms, gbs, gran = C.c_double(), C.c_double(), C.c_uint64()
        try:
            check(lib().gx_random_access_bench_alloc(gb << 30, 128, 1 << 28, 0, 2, kind, C.byref(ms),
                                                     C.byref(gbs), C.byref(gran)))
            print(json.dumps({"alloc": kind, "gib": gb, "gbs": round(gbs.value, 1),
                              "accesses_per_s": (1 << 28) / (ms.value / 1e3),
                              "granularity": gran.value}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"alloc": kind, "gib": gb, "error": str(e)}), flush=True)
