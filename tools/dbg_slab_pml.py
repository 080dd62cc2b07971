import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from test_gpu_slabs import run_single, run_group
from test_gpu_pml import channel_scene
from helpers import consistent_random_state
for variant in ("both", "pml_only", "line_only", "point"):
    s = channel_scene(32, ny=60)
    if variant == "pml_only":
        s.meta.pop("source_rows"); s.source = (40, 30)
    if variant == "line_only":
        s.meta.pop("pml")
    if variant == "point":
        s.meta.pop("pml"); s.meta.pop("source_rows"); s.source = (40, 30)
    init = consistent_random_state(s, 5)
    for n in (1, 2, 5):
        W1 = run_single(s, n, init)[0]
        W2 = run_group(s, n, init, 2, 1)[0]
        out = []
        for name, a, b in zip(("Ex", "Ey", "Hz"), W1, W2):
            d = np.argwhere(a != b)
            out.append(f"{name}: {len(d)} diffs" + (f" first {d[:6].tolist()}" if len(d) else ""))
        print(variant, n, "; ".join(out), flush=True)
