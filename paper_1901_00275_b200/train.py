"""Index.train on the GPU (reference: proj/python/bindings.cpp:44-81).

Training is outside the hot-path scope of this round (SURVEY.md §8f-1 lists
GPU training as the first "next" item).  Models trained by the reference and
exchanged as VLQ1 files (Index.load) are the supported path; this entry point
raises instead of silently training on the CPU.
"""
from __future__ import annotations


def train_model(train, k, n, m, iters, seed, clamp_lambda, device=None):
    if m == 0 or train.shape[1] % m != 0:
        raise RuntimeError("m must divide the vector dimension")
    raise RuntimeError("Index.train: GPU training is not implemented yet; load a VLQ1 model "
                       "(Index.load) trained by the reference")
