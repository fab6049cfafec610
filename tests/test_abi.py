"""CPU-side checks of the C ABI boundary: the library builds for sm_100a, loads, and exports every
symbol include/saga.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "saga.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(saga_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_00528_b200 import build
    return build.build()


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("saga_load_trace", "saga_belady_next_use", "saga_aeg_score", "saga_evict_select", "saga_replay",
              "saga_trace_info", "saga_sweep_range", "saga_comm_init", "saga_allreduce_counters", "saga_free_trace",
              "saga_comm_destroy", "saga_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_last_error_and_invalid_args_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.saga_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.saga_last_error(), bytes)
    # NULL arguments are rejected before any device work
    lib.saga_load_trace.restype = ctypes.c_int
    assert lib.saga_load_trace(None, None, 0, 0, None, None) == 1
    lib.saga_evict_select.restype = ctypes.c_int
    assert lib.saga_evict_select(None, None, None, 3, None, None, None) == 1


def test_binding_fails_loudly_without_extension(tmp_path, monkeypatch):
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "saga_copy", os.path.join(ROOT, "paper_2605_00528_b200", "saga.py"))
    mod = importlib.util.module_from_spec(spec)
    monkeypatch.setattr(os.path, "exists", lambda p: False if p.endswith("libsaga.so") else os.path.isfile(p))
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)
