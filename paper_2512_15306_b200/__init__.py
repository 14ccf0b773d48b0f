"""qtrain-b200: B200-native FP8 training step (LLMQ, arXiv 2512.15306) behind
the reference qtrain operator API.  The compute lives in libqtrain_b200.so
(hand-written sm_100a CUDA, C ABI in include/qtrain_b200.h)."""
__version__ = "0.1.0"
