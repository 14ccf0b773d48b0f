"""Stream-launched trainer step vs the same step replayed from a CUDA graph (0.5B, B=16)."""
import ctypes as C, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2512_15306_b200 import session as S, _lib
cfg = S.PRESETS["qwen2.5-0.5b"]; B, T = 16, cfg.seq_len
sess = S.Session(cfg, S.PrecisionMap(backward_grads="e5m2"), S.RunPlan(micro_batch=B), S.AdamWHyper(), seed=1234)
sess.init_params(1234)
tok = torch.from_numpy(np.random.default_rng(0).integers(0, cfg.vocab, size=B * (T + 1), dtype=np.int32)).cuda()
for i in range(3): sess.train_step(tok, B, step=i, sync=False)
sess.sync()
st = torch.cuda.ExternalStream(sess.stream)
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(10): sess.train_step(tok, B, step=3 + i, sync=False)
    e1.record(st); e1.synchronize()
    ms_stream = e0.elapsed_time(e1) / 10
    ms = C.c_float()
    rc = _lib.lib().qt_time_graph_step(sess.h, tok.data_ptr(), B * (T + 1), B, 20, 10, C.byref(ms))
    assert rc == 0
    print(f"stream {ms_stream:.2f} ms/step   graph {ms.value:.2f} ms/step", flush=True)
