"""Per-phase timing of the fused decode kernel (GR_FUSED_TIMING build).

    make -C paper_2602_22732_b200/csrc EXTRA=-DGR_FUSED_TIMING BUILD=build_timing \
        LIB=../../profiles/libgr4ad_timing.so
    GR4AD_LIB=profiles/libgr4ad_timing.so python profiles/fused_phases.py [--config c2]

Thread 0 of every CTA writes %globaltimer stamps into the workspace tail
(fused_small.cu GR_STAMP/GR_SUB); this prints the median per-CTA duration of
each phase and the CTA start/end spread (wave quantisation)."""

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2602_22732_b200.decode import BeamDecoder  # noqa: E402
from paper_2602_22732_b200.model import DecoderConfig, DecoderModel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--path", default="fused")
ap.add_argument("--batch", type=int, default=0)
args = ap.parse_args()
c = bench.CONFIGS[args.config]
cfg = DecoderConfig(*c["model"], seed=2)
B = args.batch or c["batch"]
model = DecoderModel(cfg)
dec = BeamDecoder(model, [c["S"]] * B, [list(c["widths"])] * B, path=args.path)
g = torch.Generator(device="cuda").manual_seed(0)
feats = torch.randn(B * c["S"], cfg.feat_dim, device="cuda", generator=g)
for _ in range(5):
    dec.run(features=feats)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
dec.run(features=feats)
ev[1].record()
torch.cuda.synchronize()
ws = dec.workspace
tail = ws[ws.numel() - B * 48 * 8:].view(torch.int64).view(B, 48).cpu().numpy()
t0 = tail[:, 0].min()
st = (tail - t0) / 1e3  # us
names = {0: "start", 1: "ctx proj", 2: "K/V + trunk", 4: "L0 compute", 5: "L0 select",
         6: "L1 compute", 7: "L1 select", 8: "L2 compute", 9: "L2 select", 15: "results"}
print(f"{args.config} B={B}: launch {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (events)")
print(f"CTA start spread: {np.median(st[:, 0]):.1f} us median, max {st[:, 0].max():.1f}; "
      f"end max {st[:, 15].max():.1f}")
prev = 0
order = [1, 2, 4, 5, 6, 7, 8, 9, 15]
for i in order:
    d = st[:, i] - st[:, prev]
    print(f"  {names[i]:12s} median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}")
    prev = i
if (tail[:, 16] > 0).all():
    print(f"  (trunk warp done at {np.median(st[:, 16] - st[:, 1]):.2f} us, "
          f"K/V warp 1 done at {np.median(st[:, 17] - st[:, 1]):.2f} us after ctx proj)")
tot = st[:, 15] - st[:, 0]
print(f"  per-CTA total median {np.median(tot):.1f} us")
level_start = {0: 3, 1: 5, 2: 7}
for t in range(3):
    sub = tail[:, 18 + 8 * t:26 + 8 * t]
    sub = np.where(sub > 0, sub, tail[:, [level_start[t]]])
    if True:
        s2 = (sub - tail[:, [level_start[t]]]) / 1e3
        print(f"  level-{t} warp-0 tile (fuse, ln+q, cross-attn, self+ffn, pass 1, [pass 2], window, collect)"
              f" cumulative us:", np.round(np.median(s2, 0), 2))
x = tail[:, 42:47]
if (x > 0).all():
    r = np.median((x - tail[:, [7]]) / 1e3, 0)
    print("  level-2 loop-B end (us from level start) warps 1,2,3,5,7:", np.round(r, 2),
          " window entries collected: median", np.median(tail[:, 47]), "max", tail[:, 47].max())
if os.environ.get("GR_TRUNK_STAMPS"):  # build with -DGR_NO_XSTAMP: slots 42-47 = trunk stamps
    r = np.median((tail[:, 42:48] - tail[:, [1]]) / 1e3, 0)
    print("  trunk stamps 42..47 (us after ctx proj):", np.round(r, 2))
