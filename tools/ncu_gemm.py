"""Run each small tcgen05 GEMM of the step a few times eagerly (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
import tc_bench as T  # noqa: E402  (builds the operands)

for fn in (T.head_tc, T.dA1_tc):
    for _ in range(3):
        fn()
torch.cuda.synchronize()
