"""API object model without a GPU: kinds, staging, validation, reference counts (api.py semantics)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2501_01628_b200.api import OBJECT_KINDS, Device, map_frame, render_frame_collective
from paper_2501_01628_b200.errors import UsageError
from paper_2501_01628_b200.transport import SoloEndpoint
import torch


def _device():
    return Device(SoloEndpoint(), cuda=torch.device("cuda", 0))


def test_volume_kinds_are_accepted_and_unknown_kinds_rejected():
    """Re-pointed version of the reference's test_create_rejects_unknown_kind (test_api.py:226-231):
    'volume' is now a real kind; a genuinely unknown kind is still rejected with the valid list."""
    dev = _device()
    for kind in ("volume", "spatialField", "transferFunction1D"):
        assert dev.create(kind).kind == kind
    with pytest.raises(UsageError) as err:
        dev.create("tetrahedra")
    assert "volume" in str(err.value) and "spatialField" in str(err.value)
    assert set(OBJECT_KINDS) >= {"world", "camera", "renderer", "frame"}


def test_unknown_parameter_lists_valid_names():
    cam = _device().create("camera")
    with pytest.raises(UsageError) as err:
        cam.set_param("fov", 60.0)
    assert "fovY" in str(err.value) and "aspect" in str(err.value)
    r = _device().create("renderer")
    with pytest.raises(UsageError) as err:
        r.set_param("maxDepth", 2)
    assert "ert" in str(err.value) and "composite" in str(err.value)


def test_set_param_stages_until_commit():
    dev = _device()
    sf = dev.create("spatialField")
    sf.set_param("dims", (9, 9, 9))
    sf.commit()
    sf.set_param("dims", (5, 5, 5))
    assert sf.committed["dims"] == (9, 9, 9)
    sf.commit()
    assert sf.committed["dims"] == (5, 5, 5)


def test_volume_commit_requires_committed_children():
    dev = _device()
    vol = dev.create("volume")
    with pytest.raises(UsageError, match="field"):
        vol.commit()
    sf = dev.create("spatialField")
    vol.set_param("field", sf)
    with pytest.raises(UsageError, match="field"):
        vol.commit()  # the field was never committed
    sf.commit()
    with pytest.raises(UsageError, match="transferFunction"):
        vol.commit()
    tf = dev.create("transferFunction1D")
    tf.commit()
    vol.set_param("transferFunction", tf)
    vol.commit()


def test_field_data_shape_is_validated():
    sf = _device().create("spatialField")
    sf.set_param("dims", (4, 3, 2))
    sf.set_param("data", np.zeros((2, 3, 4), np.float32))
    sf.commit()
    sf.set_param("data", np.zeros((4, 3, 2), np.float32))
    with pytest.raises(UsageError, match="does not match"):
        sf.commit()


def test_field_generators():
    sf = _device().create("spatialField")
    sf.set_param("dims", (9, 8, 7))
    sf.set_param("generator", "marschnerLobb")
    sf.set_param("frequency", 4.0)
    sf.commit()
    spec, data = sf.field_spec()
    assert data is None and spec.kind == "marschnerLobb" and spec.ml == (4.0, 0.25)
    sf.set_param("frequency", -1.0)
    with pytest.raises(UsageError, match="f_M > 0"):
        sf.commit()
    sf.set_param("generator", "noise")
    with pytest.raises(UsageError, match="unknown spatialField generator"):
        sf.commit()


def test_frame_commit_requires_children_and_size():
    dev = _device()
    frame = dev.create("frame")
    with pytest.raises(UsageError, match="world"):
        frame.commit()
    with pytest.raises(UsageError, match="before any"):
        map_frame(frame)
    with pytest.raises(UsageError, match="committed before rendering"):
        render_frame_collective(frame)


def test_world_rejects_triangle_geometry_and_empty_volumes():
    dev = _device()
    w = dev.create("world")
    w.set_param("surfaces", [dev.create("surface")])
    with pytest.raises(UsageError, match="not part of this volume path"):
        w.commit()
    w2 = dev.create("world")
    with pytest.raises(UsageError, match="exactly one"):
        w2.commit()


def test_refcounts_hold_children_until_release():
    dev = _device()
    vol = dev.create("volume")
    sf = dev.create("spatialField")
    vol.set_param("field", sf)
    assert sf.refcount == 2
    sf.release()
    assert sf.alive and sf.refcount == 1
    vol.release()
    assert not sf.alive and not vol.alive
    with pytest.raises(UsageError):
        vol.set_param("ghost", 2)
