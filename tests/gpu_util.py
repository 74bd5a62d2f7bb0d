"""Helpers for the -m gpu parity tests (host arrays <-> column-major CUDA tensors)."""
import numpy as np
import torch


def dev(a):
    """numpy (any order) -> column-major complex128 CUDA tensor."""
    if a is None:
        return None
    a = np.asfortranarray(a, dtype=np.complex128)
    return torch.from_numpy(a).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
