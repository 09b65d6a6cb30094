"""Summarise a GR4AD_PROF_DUMP file (class \\t ms \\t tag per launch, '--'
between profiled windows): mean ms per window for every (class, shape)."""
import collections
import sys

CLS = ["gemm", "attn_gemm", "topk", "softmax", "layernorm", "self_attn", "row_lse", "small",
       "collect", "fused"]
win = 0
acc = collections.OrderedDict()
for line in open(sys.argv[1]):
    line = line.rstrip("\n")
    if line == "--":
        win += 1
        continue
    c, ms, tag = line.split("\t")
    k = (CLS[int(c)], tag)
    n, t = acc.get(k, (0, 0.0))
    acc[k] = (n + 1, t + float(ms))
win = max(win, 1)
tot = sum(t for _, t in acc.values()) / win
print(f"{win} windows, {tot:.3f} ms per window")
for (c, tag), (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / win:8.3f} ms {100 * t / win / tot:5.1f}%  x{n // win:<3d} {c:10s} {tag}")
