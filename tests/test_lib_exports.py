"""The C-ABI library loads on CPU and exports every symbol include/psso.h declares."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "psso.h"
LIB = ROOT / "paper_2110_01470_b200" / "libpsso.so"


def _declared():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(psso_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_binding_list():
    from paper_2110_01470_b200 import _lib

    assert sorted(_lib.EXPORTS) == _declared()


def test_library_exports_every_declared_symbol():
    assert LIB.exists(), "run __graft_entry__.build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (psso_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version():
    from paper_2110_01470_b200 import _lib

    L = _lib.load()
    assert b"sm_100a" in L.psso_version()


def test_kernels_compiled_for_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    from paper_2110_01470_b200 import _lib

    # psso_config: 4 x int32, 4 x int64, 5 x double, uint64, double
    assert ctypes.sizeof(_lib.PssoConfig) == 16 + 32 + 40 + 8 + 8
    assert ctypes.sizeof(_lib.PssoBuffers) == 7 * 8
    cfgp = ctypes.POINTER(_lib.PssoConfig)
    L = _lib.load()
    c = _lib.PssoConfig(fn_id=5, dtype=0, nvar=128)
    assert L.psso_candidate_bytes(ctypes.byref(c)) == 32 + 128 * 8
    c32 = _lib.PssoConfig(fn_id=5, dtype=1, nvar=30)
    assert L.psso_candidate_bytes(ctypes.byref(c32)) == 32 + 128
    assert cfgp is not None


def test_invalid_config_rejected_without_device():
    """psso_create validates before touching CUDA: errors are ValueErrors with messages."""
    from paper_2110_01470_b200 import _lib

    L = _lib.load()
    ctx = ctypes.c_void_p()
    bad = _lib.PssoConfig(fn_id=5, dtype=0, rng_mode=0, nsol=10, nvar=4, row_lo=0, row_hi=10,
                          cw=0.7, cp=0.6, cg=0.8, var_min=-1, var_max=1)
    rc = L.psso_create(ctypes.byref(bad), ctypes.byref(ctx))
    assert rc == _lib.PSSO_E_INVALID
    assert "thresholds" in _lib.last_error()
    with pytest.raises(ValueError, match="thresholds"):
        _lib.check(rc)
    bad2 = _lib.PssoConfig(fn_id=4, dtype=0, nsol=10, nvar=1, row_lo=0, row_hi=10, cw=0.3,
                           cp=0.6, cg=0.8, var_min=-1, var_max=1)
    assert L.psso_create(ctypes.byref(bad2), ctypes.byref(ctx)) == _lib.PSSO_E_INVALID
    assert "f4 needs dimension" in _lib.last_error()
    bad3 = _lib.PssoConfig(fn_id=1, dtype=0, nsol=10, nvar=4, row_lo=5, row_hi=11, cw=0.3,
                           cp=0.6, cg=0.8, var_min=-1, var_max=1)
    assert L.psso_create(ctypes.byref(bad3), ctypes.byref(ctx)) == _lib.PSSO_E_INVALID
    assert "row range" in _lib.last_error()


def test_oracle_is_not_imported_by_the_product():
    pkg = ROOT / "paper_2110_01470_b200"
    for py in pkg.rglob("*.py"):
        text = py.read_text()
        assert "oracle" not in re.sub(r"#.*", "", text).replace('"""', "").lower() or \
            "import oracle" not in text, py
        assert "from oracle" not in text and "import oracle" not in text, py
    for src in list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "oracle" not in src.read_text(), src


def test_nccl_resolved_at_run_time_and_comm_arguments_checked():
    """libpsso.so has no link-time NCCL dependency: the communicator entry points
    dlopen the process's libnccl.so.2 (torch's).  No GPU needed for the unique id."""
    import subprocess

    pytest.importorskip("torch")  # loads the bundled libnccl.so.2 into the process
    from paper_2110_01470_b200 import _lib

    deps = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "libnccl" not in deps
    L = _lib.load()
    uid = (ctypes.c_ubyte * 128)()
    assert L.psso_nccl_unique_id(uid) == _lib.PSSO_OK
    assert any(bytes(uid))
    comm = ctypes.c_void_p()
    assert L.psso_comm_create(uid, 2, 2, ctypes.byref(comm)) == _lib.PSSO_E_INVALID  # rank >= nranks
    assert L.psso_comm_create(None, 1, 0, ctypes.byref(comm)) == _lib.PSSO_E_INVALID
    assert L.psso_attach_comm(None, None) == _lib.PSSO_E_INVALID
    assert L.psso_run_sharded(None, 0, 1) == _lib.PSSO_E_INVALID
    st = ctypes.c_int64()
    assert L.psso_batch_failure(ctypes.byref(st), None, None, None) == _lib.PSSO_OK and st.value == -1
