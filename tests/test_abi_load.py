"""CPU-side checks of the boundary: the library builds for sm_100a, loads without
a GPU, and exports every entry point include/co.h declares (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2204_03418_b200 import build
    return build.build()


def header_functions():
    src = open(os.path.join(ROOT, "include", "co.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return sorted(set(re.findall(r"\b(co_[a-z_]+)\s*\(", src)))


def test_header_declares_the_survey_boundary():
    fns = header_functions()
    for name in ["co_conv_create", "co_forward_step", "co_forward_steps", "co_forward", "co_state_get",
                 "co_state_set", "co_state_clean", "co_delay", "co_stack_create", "co_stack_step",
                 "co_stack_delay", "co_last_error"]:
        assert name in fns


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (co_[a-z_]+)\b", out))
    missing = [f for f in header_functions() if f not in exported]
    assert not missing, missing
    from paper_2204_03418_b200 import _abi
    assert sorted(_abi.EXPORTS) == header_functions()


def test_library_loads_without_gpu(libpath):
    L = ctypes.CDLL(libpath)
    L.co_abi_version.restype = ctypes.c_int
    assert L.co_abi_version() == 4
    L.co_last_error.restype = ctypes.c_char_p
    assert L.co_last_error() == b""


def test_sass_is_sm100a(libpath):
    """The fatbin holds sm_100a SASS (no PTX JIT, no other arch)."""
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_invalid_descriptor_is_rejected_on_host(libpath):
    """Validation happens before any CUDA call: a bad descriptor returns
    CO_ERR_ARG with a message, even on a CPU-only box."""
    from paper_2204_03418_b200 import _abi
    L = _abi.lib()
    d = _abi.CoConvDesc()
    d.spatial_rank, d.in_channels, d.out_channels, d.groups = 2, 4, 8, 3   # groups does not divide
    d.kernel = (ctypes.c_int32 * 3)(3, 3, 3)
    d.stride = (ctypes.c_int32 * 3)(1, 1, 1)
    d.dilation = (ctypes.c_int32 * 3)(1, 1, 1)
    d.in_spatial = (ctypes.c_int32 * 2)(8, 8)
    d.n_streams = 1
    h = ctypes.c_void_p()
    rc = L.co_conv_create(ctypes.byref(d), ctypes.c_void_p(1), None, 0, ctypes.byref(h))
    assert rc == _abi.CO_ERR_ARG
    assert b"groups" in L.co_last_error()
    d.groups = 1
    d.padding = (ctypes.c_int32 * 3)(3, 0, 0)                              # p_t > f - 1
    assert L.co_conv_create(ctypes.byref(d), ctypes.c_void_p(1), None, 0, ctypes.byref(h)) == _abi.CO_ERR_ARG


def test_options_api_on_host(libpath):
    """co_set_option / co_get_option / co_option_name: the documented knobs,
    their defaults, range checks and the NULL reset (host-only calls)."""
    import paper_2204_03418_b200 as co
    from paper_2204_03418_b200 import _abi
    co.reset_options()
    assert co.all_options() == _abi.OPTION_DEFAULTS
    with co.options(tc_mode=1, pair=2):
        assert co.get_option("tc_mode") == 1 and co.get_option("pair") == 2
    assert co.get_option("tc_mode") == 0 and co.get_option("pair") == 0
    with pytest.raises(_abi.CoError):
        co.set_option("no_such_option", 1)
    with pytest.raises(_abi.CoError):
        co.set_option("pair", 3)                    # out of range
    co.set_option("chunk", 0)
    co.reset_options()
    assert co.get_option("chunk") == 1


def test_release_library_reads_no_experiment_knobs(libpath):
    """The shipped library holds none of the A/B experiment variables (they are
    compiled only with -DCO_EXPERIMENTS) and no CO_* environment names at all:
    its only switches are the documented co_set_option names."""
    out = subprocess.run(["strings", libpath], capture_output=True, text=True, check=True).stdout
    leaked = sorted(set(re.findall(r"\bCO_(?:TC|PDL|CHUNK|POOL|MHA|LOG|LIB)[A-Z0-9_]*", out)))
    assert not leaked, leaked
