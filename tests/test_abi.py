"""The C-ABI boundary: libswamp_gpu.so loads, exports every entry point that
include/swamp_gpu.h declares, and the ctypes mirror matches the C layout. The
C++ facade (include/swamp/engine.hpp) compiles and links against the .so; on
a GPU it runs a case end to end."""
import ctypes as C
import json
import os
import re
import subprocess

import pytest

from paper_2206_05761_b200 import abi, gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDRS = [os.path.join(ROOT, "include", "swamp_gpu.h"), os.path.join(ROOT, "include", "swamp_io.h")]
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")


def declared_functions():
    src = "".join(open(h).read() for h in HDRS)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(swamp_(?:gpu|io|partition)_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = gpu.lib()  # loads without a GPU (cudart is static)
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(gpu.EXPORTED_SYMBOLS) == set(names)
    assert b"sm_100a" in lib.swamp_gpu_build_info()


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", gpu.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0 and "sm_100a" in out.stdout


def test_struct_layout_matches_c():
    os.makedirs(BUILD, exist_ok=True)
    src = os.path.join(BUILD, "layout.c")
    exe = os.path.join(BUILD, "layout")
    fields = [f for f, _ in abi.swamp_config._fields_]
    rfields = [f for f, _ in abi.swamp_step_report._fields_]
    with open(src, "w") as f:
        f.write('#include <stdio.h>\n#include <stddef.h>\n#include "swamp_gpu.h"\nint main(void){\n')
        f.write('printf("%zu %zu\\n", sizeof(swamp_config), sizeof(swamp_step_report));\n')
        for n in fields:
            f.write(f'printf("%zu ", offsetof(swamp_config, {n}));\n')
        f.write('printf("\\n");\n')
        for n in rfields:
            f.write(f'printf("%zu ", offsetof(swamp_step_report, {n}));\n')
        f.write('printf("\\n"); return 0; }\n')
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", exe, src])
    lines = subprocess.check_output([exe], text=True).split("\n")
    sz = list(map(int, lines[0].split()))
    assert sz == [C.sizeof(abi.swamp_config), C.sizeof(abi.swamp_step_report)]
    assert list(map(int, lines[1].split())) == [getattr(abi.swamp_config, n).offset for n in fields]
    assert list(map(int, lines[2].split())) == [getattr(abi.swamp_step_report, n).offset for n in rfields]


def _build_facade():
    os.makedirs(BUILD, exist_ok=True)
    exe = os.path.join(BUILD, "engine_facade")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-o", exe, os.path.join(ROOT, "tests", "cpp", "engine_facade.cpp"),
                           "-L", os.path.dirname(gpu.LIB_PATH), "-lswamp_gpu",
                           f"-Wl,-rpath,{os.path.dirname(gpu.LIB_PATH)}"])
    return exe


def test_cpp_facade_compiles_and_links():
    assert os.path.exists(_build_facade())


def test_config_validation_rejects_bad_input():
    # epsilon = -1 and L = 20 are rejected
    with pytest.raises(ValueError):
        abi.SimConfig(L=20, epsilon=1e-3, width=1.0).to_c()
    with pytest.raises(ValueError):
        abi.SimConfig(L=8, epsilon=-1.0, width=1.0).to_c()
    c = abi.SimConfig(L=8, epsilon=1e-3, width=40.0, t_end=3.5).to_c()
    assert c.L == 8 and c.cfl == 0.5 and c.g == 9.80665 and c.h_dry == 1e-6


@pytest.mark.gpu
def test_cpp_facade_runs_on_gpu():
    exe = _build_facade()
    out = subprocess.run([exe, "7"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout)
    assert d["t"] == 0.5 and d["covered"] == d["finest"] and d["rejected_bad_L"]
    assert abs(d["mass"] - (2.5 * 3.14159 * 2.5 ** 2 + 0.5 * (1600 - 3.14159 * 6.25))) < 2.0


@pytest.mark.gpu
def test_invalid_config_status_codes():
    import numpy as np

    cfg = abi.SimConfig(L=4, epsilon=1e-3, width=1.0)
    c = cfg.to_c()
    c.L = 20
    z = np.zeros(16 * 16)
    h = C.c_void_p()
    assert gpu.lib().swamp_gpu_create(C.byref(c), abi.dptr(z), abi.dptr(z), abi.dptr(z), abi.dptr(z), 0,
                                      C.byref(h)) == -1
    nan = np.full(16 * 16, np.nan)
    with pytest.raises(gpu.SwampError):
        gpu.initialise(cfg, nan, z, z, z)
