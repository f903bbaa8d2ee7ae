"""Mesh documents: mesh_to_json / mesh_from_json (reference cluster.hpp:95-96,
cluster.cpp:417-450) against the compiled reference (oracle/_ref): identical
canonical text for valid documents, the same error class and message for
malformed ones."""
import json

import pytest

from oracle import ref as R
from paper_2302_02599_b200 import DeviceMesh
from paper_2302_02599_b200.layout import SchemaError

needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _doc(shape, assignment=None, alpha=None, beta=None, flops=1e12):
    n = 1
    for e in shape:
        n *= e
    return json.dumps({"shape": shape,
                       "assignment": assignment if assignment is not None
                       else [f"gpu{i}" for i in range(n)],
                       "axis_alpha": alpha if alpha is not None else [2e-6] * len(shape),
                       "axis_beta_inv": beta if beta is not None else [1.1e-12] * len(shape),
                       "device_flops_per_s": flops})


@pytest.mark.parametrize("shape", [[8], [2, 4], [4, 2], [2, 2, 2], [1, 4], [3]])
def test_round_trip(shape):
    m = DeviceMesh(tuple(shape), [3e-6] * len(shape), [2e-12] * len(shape), 9.9e14)
    back = DeviceMesh.from_json(m.to_json())
    assert back == m
    assert json.loads(m.to_json())["assignment"] == [f"d{i}" for i in range(m.num_devices())]


@needs_ref
@pytest.mark.parametrize("shape", [[8], [2, 4], [2, 2, 2], [1, 4]])
def test_to_json_matches_reference_text(shape):
    m = DeviceMesh.uniform(shape)
    rc, text = R.mesh_json(m.to_json())
    assert rc == 0 and text == m.to_json()


BAD = [
    "[]",
    '"mesh"',
    json.dumps({"shape": [2]}),
    _doc([2, 0], assignment=[]),
    _doc([2, 2], assignment=["a", "b", "c"]),
    _doc([2, 2], alpha=[1e-6]),
    _doc([2, 2], beta=[1e-9, 1e-9, 1e-9]),
    json.dumps({"shape": "2x2", "assignment": [], "axis_alpha": [], "axis_beta_inv": [],
                "device_flops_per_s": 1}),
]


@needs_ref
@pytest.mark.parametrize("text", BAD)
def test_malformed_documents_raise_like_the_reference(text):
    rc, msg = R.mesh_json(text)
    assert rc == 1  # SchemaError in the reference
    with pytest.raises(SchemaError) as e:
        DeviceMesh.from_json(text)
    assert str(e.value) == msg


@needs_ref
def test_reference_documents_parse_identically():
    for shape in ([8], [2, 4], [2, 2, 2]):
        text = _doc(shape, flops=2.25e15)
        rc, canon = R.mesh_json(text)
        assert rc == 0
        m = DeviceMesh.from_json(text)
        assert m.shape == tuple(shape) and m.device_flops_per_s == 2.25e15
        assert m.axis_alpha == [2e-6] * len(shape) and m.axis_beta_inv == [1.1e-12] * len(shape)
