"""C-ABI library checks that need no GPU: the .so loads, exports every symbol
include/colgraph.h declares, and its host-only entry points behave."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "colgraph.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(\w+)\s*\([^;{]*\)\s*;", src)) - {"if", "while"})


def test_header_declares_boundary():
    names = declared_functions()
    for required in ("colgraph_build", "maxflow_solve", "mincut_extract_surface", "colgraph_free"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2601_17026_b200 import build
    lib = ctypes.CDLL(build.build())
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_names_match_abi():
    from paper_2601_17026_b200 import colgraph as cg
    for name in declared_functions():
        assert name in cg.EXPORTED, name


def test_status_strings_and_version():
    from paper_2601_17026_b200 import colgraph as cg
    for code, name in cg.STATUS.items():
        assert cg.lib().cg_status_str(code).decode() == name
    assert "sm_100a" in cg.version()


@pytest.mark.parametrize("X,nranks", [(8, 4), (7, 2), (5, 5), (512, 8), (1024, 3), (1, 1)])
def test_slab_range_partition(X, nranks):
    """Contiguous x-slabs, larger first, covering [0, X)."""
    from paper_2601_17026_b200 import colgraph as cg
    ranges = [cg.cg_slab_range(X, 4, 4, 1, r, nranks) for r in range(nranks)]
    assert ranges[0][0] == 0 and ranges[-1][1] == X
    sizes = [b - a for a, b in ranges]
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(nranks - 1))
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True) and min(sizes) >= 1


def test_slab_range_errors():
    from paper_2601_17026_b200 import colgraph as cg
    with pytest.raises(cg.ColgraphError):
        cg.cg_slab_range(3, 1, 1, 0, 0, 4)  # nranks > X  (SPEC.md TOO_MANY_SEGMENTS)
    with pytest.raises(cg.ColgraphError):
        cg.cg_slab_range(8, 1, 1, 0, 4, 4)


def test_sass_is_sm100a():
    """The shipped cubin targets sm_100a."""
    import subprocess
    from paper_2601_17026_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
