"""Debug: chained 7B stack vs layer-by-layer launches (per-layer |y|, p, v)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_14110_b200 import _capi as capi  # noqa: E402
from paper_2603_14110_b200.ffn_exec import Context, Pipeline, check  # noqa: E402
from paper_2603_14110_b200.model import build_host_model, upload  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 10
hot = int(sys.argv[2]) if len(sys.argv) > 2 else 16
cfg, host = build_host_model("7b", L, rank=256, sparsity=0.5, workers=8)
d, D = cfg["d"], cfg["D"]
layers = [upload(h, d, D, 0, 256, hot_rows=hot) for h in host]
lib = capi.lib()
arr = (C.c_void_p * L)(*[l.handle.value for l in layers])
xs = np.ascontiguousarray(np.stack([h.x for h in host]), dtype=np.float32)
for entry in ("host", "device"):
    ctx = Context(0, d, D, 256)
    ys = np.zeros_like(xs)
    st = (capi.sg_exec_stats * L)()
    if entry == "host":
        check(lib.sg_ffn_forward_layers_host(ctx.handle, arr, L, 2, xs.ctypes.data_as(C.c_void_p),
                                             ys.ctypes.data_as(C.c_void_p), 1, st, None))
    else:
        xt = torch.tensor(xs, device="cuda")
        yt = torch.zeros_like(xt)
        check(lib.sg_ffn_forward_layers(ctx.handle, arr, L, 2, C.c_void_p(xt.data_ptr()),
                                        C.c_void_p(yt.data_ptr()), 1, None))
        check(lib.sg_ctx_read_stack_stats(ctx.handle, None, L, st))
        ys = yt.cpu().numpy()
    print(entry, [(l, round(float(np.linalg.norm(ys[l])), 4), st[l].predicted_active, st[l].revalidated)
                  for l in range(L)])
# layer by layer
ctx = Context(0, d, D, 256)
x = xs[0].astype(np.float64)
out = []
for l in range(L):
    r = layers[l].forward(x, Pipeline.Sequential, ctx)
    out.append((l, round(float(np.linalg.norm(r.y)), 4), r.stats.predicted_active, r.stats.revalidated))
    x = r.y.astype(np.float32).astype(np.float64)
print("single", out)
