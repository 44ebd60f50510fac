"""CPU-side checks of the drop-in boundary: the C-ABI library exists, exports every symbol that
include/smg_b200.h declares, reports layouts consistent with the oracle, and refuses to run without
an sm_100 device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2410_09497_b200 as smg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "smg_b200.h")).read()
    return sorted(set(re.findall(r"\b(smg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = smg.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(smg.EXPORTED) == syms


@pytest.mark.parametrize("k,level", [(1, 0), (2, 3), (3, 6), (7, 5)])
def test_level_sizes_match_oracle(k, level):
    assert smg.level_sizes(k, level) == oracle.sizes(k, level)
    n = (2 << level) * (k + 1)
    assert smg.level_sizes(k, level)[4] == 3 * (n + 1) * n * n + n ** 3


def test_invalid_arguments():
    with pytest.raises(ValueError):
        smg.level_sizes(0, 1)
    with pytest.raises(ValueError):
        smg.level_sizes(1, -1)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        smg.Context(2, 2)


@pytest.mark.parametrize("k,level", [(1, 0), (2, 1)])
def test_blockvector_pressure_numbering(k, level):
    # pressure is numbered cell by cell (cells x-fastest), (k+1)^3 nodes per cell x-fastest
    H, m = k + 1, 2 << level
    n = m * H
    perm = smg.pressure_cell_local_index(k, level)
    assert sorted(perm.tolist()) == list(range(n ** 3))
    i = 0
    for cz in range(m):
        for cy in range(m):
            for cx in range(m):
                for az in range(H):
                    for ay in range(H):
                        for ax in range(H):
                            g = ((cz * H + az) * n + cy * H + ay) * n + cx * H + ax
                            assert perm[i] == g
                            i += 1
    v = np.random.default_rng(0).uniform(size=smg.level_sizes(k, level)[4])
    assert np.array_equal(smg.from_blockvector(smg.to_blockvector(v, k, level), k, level), v)


def test_dist_partition_matches_slab_partition():
    from paper_2410_09497_b200 import dist as sd
    from paper_2410_09497_b200 import slab
    for level in (2, 3, 5, 7):
        for world in (1, 2, 3, 4, 8):
            if (2 << level) < world:
                continue
            assert [sd.partition(level, world, r) for r in range(world)] == slab.partition(level, world)
