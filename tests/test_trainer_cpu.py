"""Trainer host logic (CPU): corpora and run manifests of the product trainer
(csrc/trainer.cpp) against the unmodified reference (oracle/_ref:
src/corpus.cpp, src/manifest.cpp).  The device runs (metrics, checkpoints,
resume) are in test_trainer_gpu.py."""
import json
import math

import numpy as np
import pytest

from paper_2512_15306_b200 import trainer as TR


@pytest.mark.parametrize("kind", ["perm-walk", "uniform"])
@pytest.mark.parametrize("vocab,seq,ntr,nval,seed", [(512, 128, 256, 16, 0), (151936, 64, 8, 4, 1234),
                                                     (2, 1, 1, 0, 7), (32000, 1024, 3, 2, 99)])
def test_corpus_matches_reference(ref, kind, vocab, seq, ntr, nval, seed):
    tr, va = TR.make_corpus(kind, vocab, seq, ntr, nval, seed)
    rtr, rva = ref.make_corpus(kind, vocab, seq, ntr, nval, seed)
    np.testing.assert_array_equal(tr, rtr)
    np.testing.assert_array_equal(va, rva)


def test_corpus_rejects_like_reference():
    with pytest.raises(ValueError, match="unknown corpus kind: zipf"):
        TR.make_corpus("zipf", 16, 4, 1, 1, 0)
    with pytest.raises(ValueError, match="degenerate corpus spec"):
        TR.make_corpus("uniform", 1, 4, 1, 1, 0)


def _close(a, b, path=""):
    if isinstance(a, dict):
        assert set(a) == set(b), (path, sorted(set(a) ^ set(b)))
        for k in a:
            _close(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, list):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _close(x, y, f"{path}[{i}]")
    elif isinstance(a, float) or isinstance(b, float):
        assert math.isclose(float(a), float(b), rel_tol=1e-6), (path, a, b)
    else:
        assert a == b, (path, a, b)


MANIFESTS = [
    {},
    {"seed": 7, "model": "toy", "steps": 3},
    {"seed": 11, "model": "0.5b", "precision": {"matmuls": "fp8", "backward_grads": "e5m2"},
     "plan": {"micro_batch": 16, "ga_steps": 2, "recompute": ["swiglu", "att"], "offload": "m",
              "shard_weights": True, "shard_grads": True, "lmhead_chunk_tokens": 0, "attn_chunk_rows": 128},
     "optimizer": {"lr": 3e-4, "beta2": 0.99, "weight_decay": 0.1, "max_grad_norm": 0.5, "moments": "bf16"},
     "corpus": {"kind": "uniform", "seq_len": 512, "n_train": 64, "n_val": 8, "seed": 3},
     "steps": 20, "eval_every": 5, "hardware": "h100", "workers": 8,
     "outputs": {"metrics_csv": "m.csv", "checkpoint": "c.ckpt"}},
    {"model": {"n_layers": 3, "d_model": 128, "d_ff": 512, "n_heads": 4, "n_kv_heads": 1, "vocab": 1000,
               "seq_len": 64, "tied_embeddings": True},
     "plan": {"recompute": "block", "offload": ["residuals", "theta*", "g"]}},
]


@pytest.mark.parametrize("i", range(len(MANIFESTS)))
def test_manifest_roundtrip_matches_reference(ref, i):
    text = json.dumps(MANIFESTS[i])
    _close(TR.manifest_normalize(text), ref.manifest_normalize(text))


@pytest.mark.parametrize("bad,msg", [
    ({"precision": {"matmuls": "int8"}}, "unknown matmul precision int8"),
    ({"precision": {"backward_grads": "e3m4"}}, "unknown backward grad kind e3m4"),
    ({"optimizer": {"moments": "fp16"}}, "unknown moment precision fp16"),
    ({"plan": {"recompute": ["nope"]}}, "unknown recompute site: nope"),
    ({"plan": {"offload": ["disk"]}}, "unknown offload category: disk"),
    ({"corpus": {"vocab": 7}}, "corpus vocab must match model vocab"),
    ({"corpus": {"seq_len": 4096}}, "corpus sequences longer than the model context"),
    ({"model": "70b"}, "unknown model preset '70b'"),
])
def test_manifest_errors_match_reference(ref, bad, msg):
    text = json.dumps(bad)
    with pytest.raises(ValueError, match=msg):
        TR.manifest_normalize(text)
    with pytest.raises(ref.RefError, match=msg):
        ref.manifest_normalize(text)
