"""The C++ drop-in example runs a 20-step FP8 training loop on the GPU through
the reference-named operator API and the loss goes down."""
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parent.parent


def test_cpp_example_trains(tmp_path):
    lib = ROOT / "paper_2512_15306_b200"
    exe = tmp_path / "drop_in_step"
    r = subprocess.run(["g++", "-std=c++17", "-O2", str(ROOT / "examples" / "drop_in_step.cpp"), f"-I{ROOT / 'include'}",
                        "-I/usr/local/cuda/include", f"-L{lib}", "-lqtrain_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    assert "out_of_range" in run.stdout
