"""Host logic of the peer runtime (no GPU): mesh-axis groups used by the
in-place peer all-reduce must be the reference's per-axis groups (devices
differing only on the reduced axes, mixed-radix order)."""
import itertools

import pytest

from paper_2302_02599_b200 import DeviceMesh
from paper_2302_02599_b200.peer import _group


@pytest.mark.parametrize("shape", [[8], [2, 4], [4, 2], [2, 2, 2], [2, 3]])
def test_groups_partition_the_mesh_in_mixed_radix_order(shape):
    geo = DeviceMesh.uniform(shape)
    r = len(shape)
    for k in range(1, r + 1):
        for axes in itertools.combinations(range(r), k):
            seen = set()
            for d in range(geo.num_devices()):
                g = _group(geo, d, list(axes))
                assert d in g
                size = 1
                for a in axes:
                    size *= shape[a]
                assert len(g) == size
                # ordered by the mixed-radix coordinate over `axes`
                keys = []
                for q in g:
                    c = geo.coord_of(q)
                    key = 0
                    for a in axes:
                        key = key * shape[a] + c[a]
                    keys.append(key)
                    assert all(c[a] == geo.coord_of(d)[a] for a in range(r) if a not in axes)
                assert keys == list(range(size))
                seen.add(tuple(g))
            assert sum(len(g) for g in seen) == geo.num_devices()
