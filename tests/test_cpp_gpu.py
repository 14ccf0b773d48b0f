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


def test_cpp_reference_signatures_step_and_checkpoint(tmp_path):
    """trainer.cpp:64-110 written with the reference's free-function signatures
    (build_step_context, model_forward, model_backward, global_grad_norm,
    clip_scale, adamw_step) + a QTCKPT01 save/load round trip and the
    reference's non-finite-gradient error text."""
    lib = ROOT / "paper_2512_15306_b200"
    exe = tmp_path / "ref_sig"
    r = subprocess.run(["g++", "-std=c++17", "-O2", str(ROOT / "examples" / "reference_signatures.cpp"),
                        f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include", f"-L{lib}", "-lqtrain_b200",
                        f"-Wl,-rpath,{lib}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe), str(tmp_path / "c.ckpt")], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0 and "OK" in run.stdout, run.stdout + run.stderr
