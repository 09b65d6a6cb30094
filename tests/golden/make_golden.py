"""Generate golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (~1 min)
    python tests/golden/make_golden.py --c3       # + one C3 request (~5-10 min)
    python tests/golden/make_golden.py --big      # C3 x8, C5 x8, C4-width x2 (~10 min)

Outputs (committed, read by tests/test_oracle_golden.py and the GPU parity
tests; nothing at test time reads /root/reference):

* golden_small.json  -- pre-cut instances, init checksums, beam-search
  outputs + counters on random/tiny/C1/C2 models, teacher-forced logits.
* golden_c3.json     -- one request at the C3 shape (widths 512^3).
* ref_checkpoint.npz -- (--ckpt) a checkpoint written by the reference's
  save_checkpoint, for the interop test (tests/test_api_host.py).
* golden_big.json    -- the C3 model decoded at the benched shapes:
  requests 0..7 at C3 widths 512^3, requests 0..7 at the C5 schedule
  64/128/256, and requests 0..1 at the C4 off-peak TABS widths 99/197/394
  (scale_schedule(64/128/256, 394)), each with the reference's per-level
  cut gaps (k-th minus (k+1)-th best candidate, recorded by wrapping
  beam._select) so a divergence at an intermediate level can be excused
  only where the reference's own cut was closer than tau.

Reference entry points used: adrec.serving.beam.{beam_search, topk_precut,
topk_global} (beam.py:37-143), adrec.model.decoder.{DecoderConfig,
DecoderModel, context_process, lazy_forward} (decoder.py:32-198),
adrec.model.layers.LayerCallCounter (layers.py:18-35),
adrec.verify.{random_decoder, random_context} (verify.py:83-99),
adrec.losses.supervised.fit_ecpm_buckets (supervised.py:47-76),
adrec.serving.schedule (schedule.py:33-70).
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _cfg_dict(cfg):
    return {"feat_dim": cfg.feat_dim, "d": cfg.d, "d_ff": cfg.d_ff,
            "n_layers": cfg.n_layers, "trunk_depth": cfg.trunk_depth,
            "level_vocab_sizes": list(cfg.level_vocab_sizes),
            "n_value_buckets": cfg.n_value_buckets, "seed": cfg.seed}


def params_digest(params):
    h = hashlib.sha256()
    for k, v in params.items():
        h.update(k.encode())
        h.update(np.ascontiguousarray(getattr(v, "data", v), dtype=np.float64).tobytes())
    return h.hexdigest()


def c_features(i, s_ctx, feat_dim=16):
    """Survey §8d synthetic request i."""
    return np.random.default_rng(1000 + i).normal(size=(s_ctx, feat_dim))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--big-only", action="store_true")
    ap.add_argument("--ckpt", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    from adrec.losses.supervised import fit_ecpm_buckets
    from adrec.model.decoder import (DecoderConfig, DecoderModel, context_process,
                                     lazy_forward)
    from adrec.model.layers import LayerCallCounter
    from adrec.serving import beam as ref_beam
    from adrec.serving.schedule import (BeamSchedule, TrafficSignal, resolve_dbw,
                                        scale_schedule, tabs_adjust)
    from adrec.verify import random_context, random_decoder

    def run(model, x, widths, **kw):
        counter = LayerCallCounter()
        res = ref_beam.beam_search(model, x, BeamSchedule(tuple(widths), widths[-1]),
                                   counter=counter, **kw)
        return ([list(sid.tokens) for sid, _ in res], [float(s) for _, s in res],
                [counter.layer_calls, counter.kv_builds, counter.kv_floats])

    if args.ckpt:
        # a checkpoint written by the reference's save_checkpoint (decoder.py:222-247)
        from adrec.model.decoder import save_checkpoint
        model = DecoderModel(DecoderConfig(3, 4, 6, 2, 1, (3, 3), 3, seed=123))
        save_checkpoint(model, os.path.join(HERE, "ref_checkpoint.npz"), step=17,
                        extra_arrays={"adam_t": np.array([17])}, meta={"note": "test"})
        print("wrote ref_checkpoint.npz")
        return

    if args.big or args.big_only:
        make_big(DecoderConfig, DecoderModel, context_process, ref_beam, BeamSchedule,
                 resolve_dbw, scale_schedule, run)
        if args.big_only:
            return

    out = {"generator": "tests/golden/make_golden.py", "reference": REF}

    # -- pre-cut selection (beam.py:50-89) ---------------------------------
    rng = np.random.default_rng(1)
    precut = []
    fixed = [([0.0, -1.0], [[-0.1, -2.0, -3.0], [-0.2, -0.3, -5.0]], 2),
             ([0.0, 0.0], [[-1.0, -1.0], [-1.0, -1.0]], 3),
             ([0.0], [[-1.0, -2.0]], 99)]
    for scores, lp, k in fixed:
        got = ref_beam.topk_precut([((), s) for s in scores], np.array(lp), k)
        glob = ref_beam.topk_global(scores, np.array(lp), k)
        precut.append({"scores": scores, "logprobs": lp, "k": k,
                       "expect": [[b, t, s] for b, t, s in got],
                       "expect_global": [list(map(int, glob[0])), list(map(int, glob[1])),
                                         list(map(float, glob[2]))]})
    for _ in range(300):
        b = int(rng.integers(1, 9))
        v = int(rng.integers(2, 33))
        k = int(rng.integers(1, b * v + 1))
        scores = rng.normal(size=b) * 2.0
        lp = np.log(rng.dirichlet(np.ones(v), size=b))
        got = ref_beam.topk_precut([((), float(s)) for s in scores], lp, k)
        precut.append({"scores": scores.tolist(), "logprobs": lp.tolist(), "k": k,
                       "expect": [[bb, tt, ss] for bb, tt, ss in got]})
    out["precut"] = precut

    # -- DBS integers (schedule.py:33-70) ------------------------------------
    dbs = []
    for qps, thr, slack, base, boost in [(10.0, 100.0, 1.0, 512, 0.6), (150.0, 100.0, 1.0, 512, 0.6),
                                         (100.0, 100.0, 1.0, 512, 0.6), (1.0, 10.0, 1.0, 16, 0.6),
                                         (10.0, 100.0, 0.0, 512, 0.6), (3.0, 8.0, 0.37, 8, 0.6),
                                         (1.0, 10.0, 0.5, 256, 0.6), (0.0, 5.0, 0.25, 7, 1.3)]:
        act = tabs_adjust(TrafficSignal(qps, thr, slack), base, boost)
        dbs.append({"qps": qps, "q_threshold": thr, "slack": slack, "base": base,
                    "boost": boost, "active": act})
    scaled = []
    for widths in [(4, 8, 16), (64, 128, 256), (2, 4), (1, 1, 3), (128, 256, 512)]:
        sched = resolve_dbw(list(widths), len(widths))
        for active in (sched.base_width, 26, 819, 7, 410, 1):
            scaled.append({"widths": list(widths), "active": active,
                           "expect": list(scale_schedule(sched, active).widths)})
    out["dbs"] = {"tabs": dbs, "scale": scaled}

    # -- init checksums (decoder.py:71-107) ----------------------------------
    init_cfgs = [DecoderConfig(16, 16, 32, 2, 1, (256, 256, 256), 4, seed=2),
                 DecoderConfig(3, 4, 6, 2, 1, (3, 3), 3, seed=17),
                 DecoderConfig(4, 8, 12, 3, 2, (16, 16, 16), 4, seed=0)]
    out["init"] = [{"config": _cfg_dict(c), "sha256": params_digest(DecoderModel(c).params)}
                   for c in init_cfgs]

    # -- beam search on random small models (verify.py:83-99, 400-445) -------
    beams = []
    rng = np.random.default_rng(11)
    for idx in range(40):
        model = random_decoder(rng, max_levels=3)
        feats, x = random_context(rng, model)
        sizes = model.config.level_vocab_sizes
        widths, w, reach = [], 1, 1
        for vocab in sizes:
            reach = min(reach * vocab, 64)
            w = min(max(w, int(rng.integers(1, 5))), 8, reach)
            widths.append(w)
        case = {"name": f"random{idx}", "config": _cfg_dict(model.config),
                "features": feats.tolist(), "widths": widths}
        case["tokens"], case["scores"], case["counter"] = run(model, x, widths)
        _, _, case["counter_unshared"] = run(model, x, widths, shared_kv=False)
        beams.append(case)

    def add(name, cfg, feats, widths, **kw):
        model = DecoderModel(cfg)
        x = context_process(np.atleast_2d(feats), model.params)
        case = {"name": name, "config": _cfg_dict(cfg), "widths": list(widths)}
        if "feature_request" in kw:
            case["feature_request"] = kw["feature_request"]  # c_features(i, S)
            case["s_ctx"] = int(np.asarray(feats).shape[0])
        else:
            case["features"] = np.asarray(feats).tolist()
        extra = {}
        if "trunk_depth" in kw:
            extra["trunk_depth"] = kw["trunk_depth"]
        if kw.get("value_rerank"):
            vals = np.random.default_rng(kw["bucket_seed"]).uniform(0, 3, size=50)
            buckets = fit_ecpm_buckets(vals, cfg.n_value_buckets)
            extra.update(value_rerank=True, buckets=buckets)
            case["representatives"] = [float(r) for r in buckets.representatives]
        case.update({k: v for k, v in kw.items() if k in ("trunk_depth",)})
        case["value_rerank"] = bool(kw.get("value_rerank", False))
        case["tokens"], case["scores"], case["counter"] = run(model, x, widths, **extra)
        _, _, case["counter_unshared"] = run(model, x, widths, shared_kv=False, **extra)
        beams.append(case)

    rng = np.random.default_rng(6)
    for j in range(6):
        cfg = DecoderConfig(3, 4, 6, 2, int(j % 2), (3, 3, 2), 2, seed=int(rng.integers(0, 2**31)))
        add(f"sandwich{j}", cfg, rng.normal(size=(int(rng.integers(1, 3)), 3)), (3, 9, 18))
    tiny = DecoderConfig(3, 4, 6, 2, 1, (2, 2), 3, seed=47)
    add("clamp", tiny, np.ones((1, 3)), (64, 64))
    grow = DecoderConfig(3, 6, 8, 3, 1, (4, 4, 3), 3, seed=71)
    add("grow_drop_inf", grow, np.random.default_rng(3).normal(size=(2, 3)), (1, 64, 5))
    lazy = DecoderConfig(4, 8, 12, 3, 2, (16, 16, 16), 4, seed=0)
    lazy_x = np.random.default_rng(0).normal(size=(2, 4))
    add("lazy_prog", lazy, lazy_x, (4, 8, 16))
    add("vanilla_prog", lazy, lazy_x, (4, 8, 16), trunk_depth=0)
    add("lazy_k1_override", lazy, lazy_x, (8, 8, 8), trunk_depth=1)
    rer = DecoderConfig(3, 4, 6, 2, 1, (3, 3), 3, seed=53)
    add("value_rerank", rer, np.random.default_rng(9).normal(size=(2, 3)), (3, 9),
        value_rerank=True, bucket_seed=9)
    rer0 = DecoderConfig(5, 8, 10, 3, 0, (5, 4, 3), 4, seed=59)
    add("value_rerank_k0", rer0, np.random.default_rng(19).normal(size=(3, 5)), (4, 8, 16),
        value_rerank=True, bucket_seed=19)
    wide = DecoderConfig(6, 12, 20, 4, 2, (32, 16, 64), 2, seed=5)
    add("wide_levels", wide, np.random.default_rng(23).normal(size=(7, 6)), (16, 48, 40))

    c1 = DecoderConfig(16, 16, 32, 2, 1, (256, 256, 256), 4, seed=2)
    for i in range(4):
        add(f"C1_req{i}", c1, c_features(i, 256), (32, 32, 32), feature_request=i)
    for i in range(3):
        add(f"C2_req{i}", c1, c_features(i, 256), (64, 128, 256), feature_request=i)
    out["beam"] = beams

    # -- teacher-forced logits (decoder.py:162-219) ---------------------------
    tf = []
    rng = np.random.default_rng(8)
    for idx in range(6):
        model = random_decoder(rng)
        feats = rng.normal(size=(2, model.config.feat_dim))
        x = context_process(feats, model.params)
        toks = tuple(int(rng.integers(0, v)) for v in model.config.level_vocab_sizes)
        trace = lazy_forward(model, x, toks)
        tf.append({"config": _cfg_dict(model.config), "features": feats.tolist(),
                   "tokens": list(toks),
                   "head_logits": [t.data.tolist() for t in trace.head_logits],
                   "value_logits": trace.value_logits.data.tolist()})
    out["teacher_forced"] = tf

    with open(os.path.join(HERE, "golden_small.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote golden_small.json", len(beams), "beam cases")

    if args.c3:
        cfg = DecoderConfig(16, 1024, 2048, 8, 5, (4096, 4096, 4096), 4, seed=2)
        t0 = time.time()
        model = DecoderModel(cfg)
        x = context_process(c_features(0, 1024), model.params)
        toks, scores, counter = run(model, x, (512, 512, 512))
        c3 = {"config": _cfg_dict(cfg), "request": 0, "s_ctx": 1024,
              "widths": [512, 512, 512], "init_sha256": params_digest(model.params),
              "tokens": toks, "scores": scores, "counter": counter,
              "seconds": time.time() - t0}
        with open(os.path.join(HERE, "golden_c3.json"), "w") as fh:
            json.dump(c3, fh)
        print("wrote golden_c3.json in", c3["seconds"], "s")


def make_big(DecoderConfig, DecoderModel, context_process, ref_beam, BeamSchedule,
             resolve_dbw, scale_schedule, run):
    """C3-model requests at the C3 / C5 / C4 widths, with per-level cut gaps."""
    cfg = DecoderConfig(16, 1024, 2048, 8, 5, (4096, 4096, 4096), 4, seed=2)
    model = DecoderModel(cfg)
    gaps = []
    orig = ref_beam._select

    def select(beam_scores, logprobs, k, precut):
        res = orig(beam_scores, logprobs, k, precut)
        nxt = orig(beam_scores, logprobs, k + 1, precut)[2]
        sel = res[2]
        if len(nxt) > len(sel) and len(sel) and np.isfinite(nxt[len(sel)]):
            gaps.append(float(sel[-1] - nxt[len(sel)]))
        else:
            gaps.append(None)
        return res

    ref_beam._select = select
    c4 = list(scale_schedule(resolve_dbw([64, 128, 256], 3), 394).widths)
    plan = ([("C3", i, [512, 512, 512]) for i in range(8)]
            + [("C5", i, [64, 128, 256]) for i in range(8)]
            + [("C4", i, c4) for i in range(2)])
    cases = []
    t_all = time.time()
    try:
        for name, i, widths in plan:
            t0 = time.time()
            x = context_process(c_features(i, 1024), model.params)
            del gaps[:]
            toks, scores, counter = run(model, x, widths)
            cases.append({"name": f"{name}_req{i}", "request": i, "s_ctx": 1024,
                          "widths": widths, "tokens": toks, "scores": scores,
                          "counter": counter, "level_cut_gaps": list(gaps),
                          "seconds": time.time() - t0})
            print(name, i, widths, f"{time.time() - t0:.1f}s", flush=True)
    finally:
        ref_beam._select = orig
    big = {"generator": "tests/golden/make_golden.py --big", "reference": REF,
           "config": _cfg_dict(cfg), "init_sha256": params_digest(model.params),
           "c4_widths_from": "scale_schedule(resolve_dbw([64,128,256],3), 394)",
           "cases": cases, "seconds": time.time() - t_all}
    with open(os.path.join(HERE, "golden_big.json"), "w") as fh:
        json.dump(big, fh)
    print("wrote golden_big.json in", big["seconds"], "s")


if __name__ == "__main__":
    main()
