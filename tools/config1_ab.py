"""configs[0] timing alone (bench.config1: M = 16, N = K = 4096, 24 rotating copies, one
act quant + decode launch each, PDL), diagnostics library (GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import _lib as _l  # noqa: E402
_l.use_diag_library()
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402


class A:
    pass


stream = torch.cuda.Stream()
print("config1 us:", " ".join(str(bench.config1(A(), dev, stream)["us"]) for _ in range(3)))
