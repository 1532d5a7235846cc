"""Keyed counter-based random source (reference rng.py), evaluated on the GPU.

Every deviate is a pure function of (seed, sub-stream, iteration, particle,
variable): ``u = (fold(fold(fold(mix(seed ^ stream), t), i), j) >> 11) * 2^-53``
with the SplitMix64 finalizer (rng.py:48-92).  The fused iteration kernel
regenerates exactly these bits in registers; :class:`RngStream` exposes the
same function for API parity (``psso_rng_uniform``), e.g. to count branch
events or to check the kernels' draws.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["RngStream", "SubStream"]

_MASK64 = (1 << 64) - 1


class SubStream(enum.IntEnum):
    """Independent deviate families drawn at the same (iteration, i, j) key (rng.py:34-39)."""

    BRANCH = 0x243F6A8885A308D3
    FRESH = 0x13198A2E03707344
    INIT = 0xA4093822299F31D0


@dataclass(frozen=True)
class RngStream:
    """Stateless uniform source keyed by (seed, sub-stream, iteration, particle, variable)."""

    seed: int

    def uniform(self, stream: SubStream, iteration: int, particles, variables) -> np.ndarray:
        """Uniform [0, 1) deviates at the broadcast of particle/variable indices (rng.py:73-87)."""
        import torch

        _lib.require_device()
        i, j = np.broadcast_arrays(np.asarray(particles, dtype=np.uint64),
                                   np.asarray(variables, dtype=np.uint64))
        shape = i.shape
        n = int(np.prod(shape)) if shape else 1
        it = torch.as_tensor(np.ascontiguousarray(i).reshape(-1).view(np.int64)).to("cuda")
        jt = torch.as_tensor(np.ascontiguousarray(j).reshape(-1).view(np.int64)).to("cuda")
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        rc = _lib.load().psso_rng_uniform(
            int(self.seed) & _MASK64, int(stream), int(iteration) & _MASK64, it.data_ptr(),
            jt.data_ptr(), n, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        _lib.check(rc)
        res = out.cpu().numpy().reshape(shape)
        return res if shape else np.float64(res)

    def matrix(self, stream: SubStream, iteration: int, row_lo: int, row_hi: int, nvar: int) -> np.ndarray:
        """Deviate block for particles ``row_lo..row_hi-1`` x all ``nvar`` coordinates (rng.py:89-92)."""
        i = np.arange(row_lo, row_hi, dtype=np.uint64)[:, None]
        j = np.arange(nvar, dtype=np.uint64)[None, :]
        return self.uniform(stream, iteration, i, j)
