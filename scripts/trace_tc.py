"""Timeline of the first CTA(s) of the tcgen05 kernels (needs libmonarch_b200_trace.so)."""
import ctypes
import os
import sys

os.environ["MBX_LIB"] = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2602_12271_b200",
                                     "libmonarch_b200_trace.so")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_12271_b200 import _lib, ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "sf"
wl = bench.workload(cfg, 1)
dev = torch.device("cuda", 0)
q = torch.randn(wl["B"], wl["H"], wl["nq"], wl["d"], device=dev, dtype=torch.bfloat16)
k = torch.randn(wl["B"], wl["H"], wl["nk"], wl["d"], device=dev, dtype=torch.bfloat16)
v = torch.randn(wl["B"], wl["H"], wl["nk"], wl["dv"], device=dev, dtype=torch.bfloat16)
lib = _lib.load()
lib.mbx_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
buf = np.zeros(4 * 16 * 2048, dtype=np.uint64)
lib.mbx_trace_col_dump.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
bufc = np.zeros(4 * 16 * 2048, dtype=np.uint64)
for it in range(3):
    ops.forward(q, k, v, wl["low"], 1)
    torch.cuda.synchronize()
    lib.mbx_trace_dump(buf.ctypes.data, buf.nbytes)   # keep only the last run's trace
    lib.mbx_trace_col_dump(bufc.ctypes.data, bufc.nbytes)
ev = buf.reshape(4, 16, 2048)
lib.mbx_span_dump.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
span = np.zeros(2 * 256 * 2, dtype=np.uint64)
lib.mbx_span_dump(span.ctypes.data, span.nbytes)
span = span.reshape(2, 256, 2).astype(np.int64)
t0s = span[0, :, 0][span[0, :, 0] > 0].min()
for kern, name in ((0, "row"), (1, "col")):
    ok = span[kern, :, 0] > 0
    if not ok.any():
        continue
    st = (span[kern, ok, 0] - t0s) / 1000.0
    en = (span[kern, ok, 1] - t0s) / 1000.0
    print(f"span {name}: ctas {ok.sum()} start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} "
          f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
    print("  ends:", " ".join(f"{x:.1f}" for x in np.sort(en)[:: max(1, len(en) // 24)]))
for cta in range(int(os.environ.get("NCTA", "1"))):
    allt = [int(x) >> 8 for x in ev[cta].ravel() if x]
    t0 = min(allt) if allt else 0
    for role in range(16):
        xs = [(int(x) >> 8, int(x) & 255) for x in ev[cta, role] if x]
        if not xs:
            continue
        print(f"cta {cta} role {role}: {len(xs)} events")
        print("  " + " ".join(f"{tag}@{(t - t0) / 1000:.2f}" for t, tag in xs[:160]))

evc = bufc.reshape(4, 16, 2048)
for cta in range(int(os.environ.get("NCTA", "1"))):
    allt = [int(x) >> 8 for x in evc[cta].ravel() if x]
    if not allt:
        continue
    for role in range(16):
        xs = [(int(x) >> 8, int(x) & 255) for x in evc[cta, role] if x]
        if not xs:
            continue
        print(f"col cta {cta} role {role}: {len(xs)} events")
        print("  " + " ".join(f"{tag}@{(t - t0s) / 1000:.2f}" for t, tag in xs[:200]))
