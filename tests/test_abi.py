"""CPU checks of the C-ABI boundary (no compute calls without a GPU):
the library loads, exports every symbol include/distir.h declares, the
ctypes layouts match the header's struct sizes, and the host-side shard
planner partitions the index space."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "distir.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(distir_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2111_05426_b200 as pkg
    declared = _header_functions()
    assert set(declared) == set(pkg.EXPORTS)
    so = ctypes.CDLL(pkg.SO_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert pkg.distir_version().startswith("distir-b200")


def test_library_is_sm100a():
    import subprocess
    import paper_2111_05426_b200 as pkg
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    import paper_2111_05426_b200 as pkg
    assert ctypes.sizeof(pkg.distir_config) == 32
    assert ctypes.sizeof(pkg.distir_topk_entry) == 32
    assert ctypes.sizeof(pkg.distir_model) == 52      # 13 x int32
    assert ctypes.sizeof(pkg.distir_topology) == 120
    assert pkg.TOPK_DTYPE.itemsize == 32


@pytest.mark.parametrize("n,G", [(0, 1), (1, 1), (7, 3), (8680, 8), (20, 4),
                                 (5, 8), (1000003, 7)])
def test_shard_planner_partitions(n, G):
    import paper_2111_05426_b200 as pkg
    seen = np.zeros(n, dtype=np.int64)
    sizes = []
    for g in range(G):
        idx = pkg.distir_shard_indices(n, g, G)
        assert (np.diff(idx) > 0).all()
        seen[idx] += 1
        sizes.append(len(idx))
    assert (seen == 1).all()
    assert max(sizes) - min(sizes) <= 1


def test_errors_do_not_abort():
    """Invalid arguments come back as status codes, not crashes."""
    import paper_2111_05426_b200 as pkg
    h = ctypes.c_void_p()
    st = pkg.lib.distir_sim_create(None, 0, None, 0, 0, None, ctypes.byref(h))
    assert st == 1 and "models" in pkg.lib.distir_last_error().decode()
    st = pkg.lib.distir_grid_size(None, None, None)
    assert st == 1
