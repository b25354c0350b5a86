"""paper_2311_09550_b200 -- B200-native (sm_100a) W4A8 FastGEMM linear layer.

The drop-in for the reference's FastGEMM hot path (OdysseyLLM, arXiv 2311.09550):
per-token INT8 activation quantization, per-channel INT4 weight packing, the
W4A8 GEMM with the SINT4->S8 high-nibble widening, and the dequantizing epilogue,
all as hand-written CUDA for sm_100a behind a C ABI (include/odyssey_b200.h).

Submodules:
    api     -- host-buffer mirror of the reference interface (numpy in / out)
    device  -- stream-ordered device API on torch tensors, W4A8Linear
    tp      -- Megatron-style column/row-parallel W4A8 linears (torch.distributed)
"""
from ._lib import OdyError, build_library, lib  # noqa: F401

__all__ = ["OdyError", "build_library", "lib", "api", "device", "tp"]
