"""The C-ABI library loads on a CPU host and exports every symbol include/tdb.h declares."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "tdb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tdb_\w+)\s*\(", src, re.M)))


def test_header_symbols_exported():
    from paper_1503_07221_b200 import _lib

    names = declared()
    assert len(names) >= 15
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTED)
    assert _lib.LIB.tdb_abi_version() == 1


def test_no_device_errors_are_loud():
    from paper_1503_07221_b200 import _lib

    if _lib.device_count() > 0:
        return
    import pytest

    with pytest.raises(RuntimeError):
        _lib.Context(0)


def test_library_resolves_every_symbol_at_load():
    # RTLD_NOW: an internal symbol declared in a header but left undefined (e.g. defined
    # inside an anonymous namespace) fails here instead of on the GPU box
    from paper_1503_07221_b200 import _lib

    ctypes.CDLL(_lib.LIB_PATH, mode=os.RTLD_NOW)


def test_ctypes_structs_match_the_header(tmp_path):
    # the ctypes mirrors in _lib.py must have the size and field offsets of include/tdb.h
    # (a C program compiled against the header prints them)
    import shutil
    import subprocess

    import pytest

    from paper_1503_07221_b200 import _lib

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "sizes.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "tdb.h"\n'
        "int main(void) {\n"
        '  printf("%zu %zu %zu %zu\\n", sizeof(TdbStats), offsetof(TdbStats, ms_quad_cells),\n'
        "         offsetof(TdbStats, n_in_cells), offsetof(TdbStats, pairs_cells));\n"
        '  printf("%zu %zu\\n", sizeof(TdbPsiPack), sizeof(TdbMatvecDesc));\n'
        "  return 0;\n}\n"
    )
    exe = tmp_path / "sizes"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    size, o_ms, o_nin, o_pairs, size_pack, size_mv = (int(v) for v in out)
    S = _lib.TdbStats
    assert ctypes.sizeof(S) == size
    assert (S.ms_quad_cells.offset, S.n_in_cells.offset, S.pairs_cells.offset) == (o_ms, o_nin, o_pairs)
    assert ctypes.sizeof(_lib.TdbPsiPack) == size_pack
    assert ctypes.sizeof(_lib.TdbMatvecDesc) == size_mv
