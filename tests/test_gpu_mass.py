"""The GPU mass function of the mass-weighted kd split (device.field_mass_function) equals the host
restatement on the oracle's voxels, box for box, and drives decompose() to the same bricks."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2501_01628_b200 import device as dev
from paper_2501_01628_b200.volume import blob_field, decompose

pytestmark = pytest.mark.gpu


def _host_mass(vox, tau):
    mask = (vox >= tau).astype(np.int64)

    def mass(axis, lo, hi):
        sub = mask[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        return sub.sum(axis=tuple(a for a in range(3) if a != 2 - axis))

    return mass


@pytest.mark.parametrize("chunk", [5, 64])
def test_field_mass_function_matches_host(cuda_device, oracle_lib, chunk):
    f = blob_field((41, 37, 34), seed=6, n_blobs=8, lopsided=True)
    vox = oracle.generate_field(f.dims, f.blobs)
    want = _host_mass(vox, 0.1)
    got = dev.field_mass_function(f, cuda_device, 0.1, chunk=chunk)
    for axis in range(3):
        for lo, hi in [((0, 0, 0), (40, 36, 33)), ((3, 5, 7), (29, 30, 21)), ((10, 0, 0), (11, 36, 33))]:
            assert np.array_equal(got(axis, lo, hi), want(axis, lo, hi)), (axis, lo, hi)
    for P in (2, 3, 8):
        assert decompose(f, P, "mass", got).boxes == decompose(f, P, "mass", want).boxes
