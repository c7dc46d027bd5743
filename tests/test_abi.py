"""The C ABI: libpgx.so loads without a GPU and exports every symbol include/pgx.h declares."""

import ctypes
import os
import subprocess

import pytest

from paper_1706_00095_b200 import _lib


def test_library_is_built():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"


def test_every_header_symbol_is_exported_and_bound():
    declared = _lib.header_symbols()
    assert len(declared) >= 30
    handle = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(handle, name), f"{name} declared in pgx.h but not exported"
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signature table drifted from pgx.h"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported


def test_abi_version_and_error_channel():
    lib = _lib.lib()
    assert lib.pgx_abi_version() == 3
    assert isinstance(_lib.last_error(), str)


def test_built_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_means_a_loud_error_not_a_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    rc = _lib.lib().pgx_world_create(0, 1, 0, ctypes.byref(h))
    assert rc != 0
    with pytest.raises(Exception):
        _lib.call("pgx_world_create", 0, 1, 0, ctypes.byref(h))


def test_product_path_never_imports_the_oracle():
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1706_00095_b200")
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "from oracle" not in src and "import oracle" not in src


def test_header_constants_match_the_python_mirror():
    """Enum values and limits in include/pgx.h are what _lib / exchange / errors use."""
    import re

    from paper_1706_00095_b200 import errors
    from paper_1706_00095_b200.exchange import FLAGS, MODES, VARIANT_ALIASES, VARIANTS

    text = open(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "include", "pgx.h")).read()
    enum = {m.group(1): int(m.group(2)) for m in re.finditer(r"\b(PGX_[A-Z0-9_]+)\s*=\s*(\d+)", text)}
    define = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+(PGX_[A-Z0-9_]+)\s+(\d+)", text)}
    for name, val in VARIANTS.items():
        if name in VARIANT_ALIASES:  # a library variant run with a flag
            base, flag = VARIANT_ALIASES[name]
            assert VARIANTS[base] == val and flag in FLAGS, name
            continue
        assert enum["PGX_VARIANT_" + name.upper()] == val, name
    for name, val in FLAGS.items():
        assert enum["PGX_XF_" + name.upper()] == val, name
    for name, val in MODES.items():
        assert enum["PGX_MODE_" + name.upper()] == val, name
    assert define["PGX_XCHG_STREAMS"] == _lib.XCHG_STREAMS
    assert define["PGX_CKPT_MAX_LAYERS"] == _lib.CKPT_MAX_LAYERS
    assert define["PGX_MAX_RANKS"] == _lib.MAX_RANKS
    assert define["PGX_MAX_PIECES"] == _lib.MAX_PIECES
    assert define["PGX_IPC_HANDLE_BYTES"] == _lib.IPC_HANDLE_BYTES
    status = {k[len("PGX_E_"):]: v for k, v in enum.items() if k.startswith("PGX_E_")}
    assert set(errors.STATUS_CLASSES) == set(status.values())
    assert errors.STATUS_CLASSES[status["FORMAT"]] is errors.FormatError
    assert errors.STATUS_CLASSES[status["TIMEOUT"]] is errors.TransportError
