"""Profiling aid: cProfile of ServingEngine.serve_batch on the C2 model (128-request
batches after warm-up) with the callers of torch.cuda.is_available / Stream.__new__."""
import cProfile, pstats, sys, os, numpy as np
sys.path.insert(0, os.getcwd())
import torch
from paper_2602_22732_b200.model import DecoderConfig, DecoderModel
from paper_2602_22732_b200.serving import BeamSchedule, ServingConfig, ServingEngine, SnapshotStore
from paper_2602_22732_b200.quantizer import SidIndex
model = DecoderModel(DecoderConfig(16, 16, 32, 2, 1, (256,)*3, 4, seed=2))
eng = ServingEngine(SnapshotStore(model), SidIndex(), ServingConfig(BeamSchedule((64,128,256),256), q_threshold=1e9))
f = [np.random.default_rng(i).normal(size=(256, 16)) for i in range(128)]
eng.warmup(f[0], 128)
k = [0]
def go():
    for it in range(40):
        reqs = [(f"u{k[0]}_{i}", f[i], it * 0.01) for i in range(128)]
        k[0] += 1
        eng.serve_batch(reqs, it * 0.01)
go()
pr = cProfile.Profile(); pr.enable(); go(); pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
st.print_callers("is_available")
st.print_callers("__new__")
