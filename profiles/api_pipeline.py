"""beam_search_batch (the drop-in API) at C3 / C5 bench shapes with 1-4
pipelined request groups: serial calls, host float64 features in, result
lists out (the bench's e2e_api measurement, per group count)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2602_22732_b200.model import DecoderConfig, DecoderModel  # noqa: E402
from paper_2602_22732_b200.serving import beam_search_batch  # noqa: E402

for name in sys.argv[1:] or ["c5", "c3"]:
    c = bench.CONFIGS[name]
    model = DecoderModel(DecoderConfig(*c["model"], seed=2))
    B, S = c["batch"], c["S"]
    feats = [np.random.default_rng(1000 + i).normal(size=(S, c["model"][0])) for i in range(B)]
    sched = [tuple(c["widths"])] * B
    for parts in (1, 2, 3, 4):
        for _ in range(2):
            beam_search_batch(model, features=feats, schedules=sched, pipeline=parts)
        reps = 4
        t0 = time.perf_counter()
        for _ in range(reps):
            beam_search_batch(model, features=feats, schedules=sched, pipeline=parts)
        dt = (time.perf_counter() - t0) / reps
        print(f"{name} pipeline={parts}: {1e3 * dt:.1f} ms per call, {B / dt:.0f} req/s", flush=True)
