"""B200-native VLQ-ADC search engine (arXiv 1901.00275).

The product is ``libvlqgpu.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/vlq_gpu.h``); ``paper_1901_00275_b200.vlqadc`` is the drop-in
mirror of the reference's ``vlqadc`` Python module on top of it.
"""
from . import vlqadc  # noqa: F401

__all__ = ["vlqadc"]
