"""Helpers for the gpu-marked parity tests (inputs to the device, tolerance checks)."""
import numpy as np


def dev_coo(t):
    import torch
    ind = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()
           for a in t.ind]
    vals = torch.from_numpy(np.ascontiguousarray(t.vals, dtype=np.float64)).cuda()
    return ind, vals


def dev_factors(F, ld=None, pad_value=0.0):
    """Factors as CUDA tensors with leading dimension ld (pad columns = pad_value)."""
    import torch
    out = []
    for A in F:
        I, R = A.shape
        L = ld or R
        B = np.full((I, L), pad_value)
        B[:, :R] = A
        out.append(torch.from_numpy(B).cuda())
    return out


def rel_fro(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b.ravel())
    return np.linalg.norm((a - b).ravel()) / (nb if nb > 0 else 1.0)


# BASELINE.json north star tolerances.
MTTKRP_TOL = 1e-10
ALS_TOL = 1e-7
