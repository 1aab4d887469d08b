"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/rbicg.h declares (no compute calls without a GPU)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "rbicg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rbicg_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1010_0762_b200 import _lib
    names = header_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(_lib.lib, name), name
        assert name in _lib.EXPORTED, name


def test_strerror_and_invalid_args_without_gpu():
    import ctypes as C
    from paper_1010_0762_b200 import _lib
    assert _lib.lib.rbicg_strerror(0) == b"ok"
    assert _lib.lib.rbicg_strerror(-5).startswith(b"LAPACK")
    # NULL handles are rejected before any CUDA call
    assert _lib.lib.rbicg_solve_dual(None, None, None, None, None, None, None,
                                     None, None, 0, None, None) == -1
    assert _lib.lib.rbicg_init(None, 0, None, None) == -1


def test_struct_layouts_match_header():
    import ctypes as C
    from paper_1010_0762_b200 import _lib
    assert C.sizeof(_lib.Opts) == 4 * 3 + 4 + 8 * 2 + 8 + 4 * 4
    assert C.sizeof(_lib.Result) == 5 * 4 + 4 + 8 * 10 + 8
    assert C.sizeof(_lib.Dist) == 4 + 4 + 128 + 8 + 8 + 4 + 4


def test_opts_field_order_matches_header():
    """rbicg_opts fields in header order (include/rbicg.h), ending with
    `pencil` (the §4.4 switch) at the last 4-byte slot."""
    import re
    import ctypes as C
    from pathlib import Path
    from paper_1010_0762_b200 import _lib
    hdr = (Path(__file__).resolve().parents[1] / "include" / "rbicg.h").read_text()
    body = hdr[:hdr.index("} rbicg_opts;")]
    body = body[body.rindex("typedef struct {"):]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"\b(?:int32_t|uint64_t|double)\s+(\w+);", body)
    assert names == [f for f, _ in _lib.Opts._fields_]
    assert _lib.Opts.pencil.offset == C.sizeof(_lib.Opts) - 4
