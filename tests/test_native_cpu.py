"""The native library without a GPU: it loads, exports every entry point the
C-ABI header declares, and its host-side logic matches the reference; no
compute path ever runs on the CPU."""
import ctypes
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "qtrain_b200.h"
LIB = ROOT / "paper_2512_15306_b200" / "libqtrain_b200.so"


def _declared():
    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(qtk?_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "build the library first (python __graft_entry__.py)"
    lib = ctypes.CDLL(str(LIB))
    names = _declared()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_sm100a_code_only():
    """cubins in the library are sm_100a with tcgen05 / TMA instructions."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    for mnem in ("UTCQMMA", "UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem


def test_shard_layout_and_streams_match_reference_rules():
    from oracle import port
    from paper_2512_15306_b200 import session as S
    for n in (1, 255, 256, 1000, 3000, 136_134_656):
        for w in (1, 2, 3, 4, 8):
            assert S.shard_layout(n, w) == port.shard_layout(n, w)
    for name in ("gradaccum/embed", "adamw/layers.0.w_qkv/m", "init/lm_head"):
        assert S.fnv1a64(name) == port.fnv1a64(name)


def test_no_cpu_fallback():
    """Without a CUDA device the session refuses to run (fails loudly)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2512_15306_b200 import session as S
    with pytest.raises(Exception):
        S.Session(S.ModelConfig(), plan=S.RunPlan(micro_batch=1))


def test_ops_reject_cpu_tensors():
    import torch
    from paper_2512_15306_b200 import ops
    with pytest.raises(ValueError, match="CUDA"):
        ops.absmax(torch.zeros(8, dtype=torch.bfloat16))


def test_flops_accounting_matches_reference(ref):
    from paper_2512_15306_b200 import session as S
    for name in ("qwen2.5-0.5b", "qwen2.5-1.5b", "qwen2.5-14b"):
        c = S.PRESETS[name]
        a, b = ref.flops_per_token(c.as_list())
        fp8, bf16 = c.flops_per_token()
        assert abs(fp8 - a) / a < 1e-12 and abs(bf16 - b) / b < 1e-12


def test_cpp_drop_in_header_compiles(tmp_path):
    """The C++ operator-API header (include/qtrain_b200/qtrain.hpp) and the
    example compile against the library with g++."""
    import subprocess
    exe = tmp_path / "drop_in_step"
    r = subprocess.run(["g++", "-std=c++17", "-O1", str(ROOT / "examples" / "drop_in_step.cpp"), f"-I{ROOT / 'include'}",
                        "-I/usr/local/cuda/include", f"-L{LIB.parent}", "-lqtrain_b200",
                        f"-Wl,-rpath,{LIB.parent}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
