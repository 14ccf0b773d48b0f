"""Python mirror of the trainer C ABI (csrc/trainer.cpp): corpora, run
manifests, the manifest-driven device trainer and QTCKPT01 checkpoints.

Names follow the reference (src/corpus.cpp make_corpus, src/manifest.cpp
manifest_from_json / manifest_to_json, src/trainer.cpp run_training_to_files,
src/checkpoint.cpp save_checkpoint / load_checkpoint).
"""
from __future__ import annotations

import ctypes as C
import json
import struct

import numpy as np

from . import session as S

_vp, _i64, _u64, _ci = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
_SIGS = {
    "qt_train_last_error": (C.c_char_p, []),
    "qt_make_corpus": (_ci, [C.c_char_p, _i64, _ci, _ci, _ci, _u64, _vp, _vp]),
    "qt_manifest_normalize": (_ci, [C.c_char_p, _vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "qt_run_training": (_ci, [C.c_char_p, _ci, _vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "qt_checkpoint_save": (_ci, [C.POINTER(_vp), _ci, C.POINTER(S._Cfg), C.c_char_p, _ci]),
    "qt_checkpoint_load": (_ci, [C.POINTER(_vp), _ci, C.c_char_p, C.POINTER(_i64)]),
}
_bound = None


def _lib():
    global _bound
    if _bound is None:
        from . import _lib as L
        l = L.lib()
        for n, (rt, at) in _SIGS.items():
            f = getattr(l, n)
            f.restype = rt
            f.argtypes = at
        _bound = l
    return _bound


def _chk(rc: int) -> None:
    if rc == 0:
        return
    msg = _lib().qt_train_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _text(fn, *args) -> str:
    need = C.c_size_t(0)
    _chk(fn(*args, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _chk(fn(*args, buf, need.value, C.byref(need)))
    return buf.value.decode()


def make_corpus(kind: str, vocab: int, seq_len: int, n_train: int, n_val: int, seed: int):
    """(train, val) flattened (seq_len + 1)-token sequences (src/corpus.cpp:58-69)."""
    tr = np.empty(n_train * (seq_len + 1), np.int32)
    va = np.empty(max(n_val, 0) * (seq_len + 1), np.int32)
    _chk(_lib().qt_make_corpus(kind.encode(), vocab, seq_len, n_train, n_val, seed, tr.ctypes.data,
                               va.ctypes.data if va.size else None))
    return tr, va


def manifest_normalize(manifest: str | dict) -> dict:
    """manifest_to_json(manifest_from_json(...)) of a manifest (JSON text, dict or path)."""
    text = json.dumps(manifest) if isinstance(manifest, dict) else manifest
    return json.loads(_text(_lib().qt_manifest_normalize, text.encode()))


def run_training(manifest: str | dict, device_count: int = 0) -> dict:
    """run_training_to_files on the device (metrics CSV + checkpoint per the manifest's
    outputs); returns {"metrics": [...], "initial_train_loss", "final_train_loss", ...}."""
    text = json.dumps(manifest) if isinstance(manifest, dict) else manifest
    return json.loads(_text(_lib().qt_run_training, text.encode(), device_count))


def save_checkpoint(sessions, path: str, with_optimizer: bool = True) -> None:
    ss = sessions if isinstance(sessions, (list, tuple)) else [sessions]
    arr = (_vp * len(ss))(*[s.h for s in ss])
    cfg = S._Cfg(*ss[0].cfg.as_list())
    _chk(_lib().qt_checkpoint_save(arr, len(ss), C.byref(cfg), path.encode(), int(with_optimizer)))


def load_checkpoint_into(sessions, path: str) -> int:
    """Params (+ moments and step count when present) from a QTCKPT01 file into the
    sessions; returns the optimizer step it continues from."""
    ss = sessions if isinstance(sessions, (list, tuple)) else [sessions]
    arr = (_vp * len(ss))(*[s.h for s in ss])
    st = _i64(0)
    _chk(_lib().qt_checkpoint_load(arr, len(ss), path.encode(), C.byref(st)))
    return st.value


def read_checkpoint(path: str) -> tuple[dict, dict]:
    """Parse a QTCKPT01 file (src/checkpoint.cpp:19-80): (manifest, {name: f32 array})."""
    with open(path, "rb") as f:
        blob = f.read()
    if blob[:8] != b"QTCKPT01":
        raise RuntimeError(f"not a checkpoint file: {path}")
    (n,) = struct.unpack_from("<Q", blob, 8)
    man = json.loads(blob[16:16 + n].decode())
    base = 16 + n
    out = {}
    for e in man["tensors"]:
        off = base + 4 * e["offset_elems"]
        out[e["name"]] = np.frombuffer(blob, np.float32, e["numel"], off).reshape(e["shape"])
    return man, out
