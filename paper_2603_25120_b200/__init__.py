"""paper_2603_25120_b200 -- B200-native DFLOP plan-candidate evaluator (arXiv 2603.25120).

The compute path is the C-ABI library ``libdflop.so`` (hand-written sm_100a CUDA,
``csrc/``), declared in ``include/dflop.h``; ``dflop`` is its thin ctypes binding.
There is no CPU fallback: importing ``paper_2603_25120_b200.dflop`` without the built
library raises.
"""
__all__ = ["synth", "dflop"]
