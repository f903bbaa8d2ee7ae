"""tools/pair_sweep.py claims "every spec-to-spec conversion": its spec
enumeration must be exactly the reference's (enumerate_specs, layout.cpp,
via oracle/_ref) for the swept meshes and tensors (CPU)."""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))


@pytest.mark.parametrize("mesh,shape", [([2, 4], (8192, 8192)), ([2, 2, 2], (8192, 8192)),
                                        ([2, 2, 2], (512, 512, 256)), ([8], (65536, 8192))])
def test_pair_sweep_enumerates_the_reference_specs(mesh, shape):
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    from pair_sweep import specs

    mine = specs(len(shape), len(mesh), shape, mesh)
    theirs = sorted(ref.all_valid_specs(mesh, shape, 2))
    assert mine == theirs
