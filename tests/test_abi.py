"""The C-ABI library loads without a GPU and exports every symbol declared in
include/sk_stencil.h (no compute calls here)."""
from __future__ import annotations

import ctypes

import pytest

from paper_1511_02490_b200 import _native as N


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = N.header_symbols()
    assert len(syms) >= 10
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"


def test_prototypes_cover_header():
    assert set(N.header_symbols()) == set(N._PROTOTYPES)


def test_descriptor_layout_matches_header():
    # int32 x7 (+4 pad), double at 32, int32 x5 (+4 pad) -> 64 bytes
    assert ctypes.sizeof(N.sk_stencil_desc) == 64
    assert N.sk_stencil_desc.pad_value.offset == 32


def test_version_and_error_strings():
    assert N.lib().sk_version().decode().startswith("sk_stencil")
    assert isinstance(N.last_error(), str)


def test_fill_host_matches_reference_rng():
    # uniform01 = (mt19937_64() >> 11) * 2^-53 (rng.hpp:48) -> kind 1 (float64)
    import numpy as np

    from paper_1511_02490_b200 import fill_host

    a = np.empty(5, np.float64)
    fill_host(a, 1, 5489)
    # std::mt19937_64 default seed 5489: first output 14514284786278117030
    assert a[0] == (14514284786278117030 >> 11) * 2.0 ** -53


def test_fill_host_equals_oracle_fill():
    # the bench's GPU arm fills through the product library, the reference
    # arm through oracle_fill: the two streams must be identical
    import numpy as np

    import oracle_lib as O
    from paper_1511_02490_b200 import fill_host

    for dtype in ("int32", "float32", "float64"):
        for kind in range(4):
            a = np.empty((37, 41), dtype)
            fill_host(a, kind, 1000 + kind)
            assert a.tobytes() == O.fill((37, 41), dtype, kind, 1000 + kind).tobytes()


def test_invalid_descriptor_is_einval_without_gpu():
    d = N.sk_stencil_desc(op=99, dtype=1)
    km = ctypes.c_int32(0)
    rc = N.lib().sk_kernel_max_wgsize(ctypes.byref(d), ctypes.byref(km))
    assert rc == N.SK_EINVAL


@pytest.mark.parametrize("field,value", [("dtype", 7), ("border_mode", 3), ("north", 65),
                                         ("load_path", 9)])
def test_bad_fields_rejected(field, value):
    d = N.sk_stencil_desc(op=0, dtype=1, north=1, south=1, east=1, west=1)
    setattr(d, field, value)
    rc = N.lib().sk_stencil_launch(ctypes.byref(d), 1, 1, 8, 8, 8, 8, 0, 0, 2, 2, None)
    assert rc == N.SK_EINVAL


def test_wgtb_c_api_exports():
    """libwgtb exports every function include/wgtb_c.h declares."""
    import re

    from paper_1511_02490_b200 import autotune
    lib = autotune.lib()
    header = (N.REPO_ROOT / "include" / "wgtb_c.h").read_text()
    names = set(re.findall(r"^(?:int|void|const char\*)\s+(wgtb_\w+)\(", header, re.M))
    assert {"wgtb_predict", "wgtb_shortlist", "wgtb_tune_measured", "wgtb_launch_tuned"} <= names
    for n in names:
        assert hasattr(lib, n), n
