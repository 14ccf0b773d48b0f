"""Run W warm-up trainer steps, then ONE step inside cudaProfilerStart/Stop so
`ncu --profile-from-start off` captures exactly one step's launches.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python scripts/profile_step.py --config qwen2.5-0.5b
"""
import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2512_15306_b200 import session as S

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="qwen2.5-0.5b")
ap.add_argument("--micro-batch", type=int, default=16)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--recompute", default="")
ap.add_argument("--ga", type=int, default=1, help="micro-batches per step (the bench default accumulates ~500k tokens)")
args = ap.parse_args()
cfg = S.PRESETS[args.config]
B, T = args.micro_batch, cfg.seq_len
plan = S.RunPlan(micro_batch=B, ga_steps=args.ga, recompute=tuple(x for x in args.recompute.split(",") if x))
sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), plan, S.AdamWHyper(), seed=1234)
sess.init_params(1234)
tok = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, size=args.ga * B * (T + 1), dtype=np.int32)).cuda()
for i in range(args.warmup):
    sess.train_step(tok, B, step=i, sync=False)
sess.sync()
torch.cuda.profiler.start()
sess.train_step(tok, B, step=args.warmup, sync=False)
sess.sync()
torch.cuda.profiler.stop()
print("profiled one step")
