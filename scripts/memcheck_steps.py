"""A few trainer steps (stream + graph replay) at small shapes, for compute-sanitizer runs."""
import pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_15306_b200 import session as S
for cfg in (S.ModelConfig(2, 128, 256, 2, 1, 256, 128), S.ModelConfig(2, 256, 512, 2, 2, 304, 128)):
    sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), S.RunPlan(micro_batch=2, ga_steps=2), seed=5)
    sess.init_params(5)
    for st in range(3):
        toks = np.random.default_rng(st).integers(0, cfg.vocab, size=2 * 2 * (cfg.seq_len + 1), dtype=np.int32)
        print(cfg.d_model, st, sess.train_step(toks, 2, step=st))
