"""C-ABI boundary checks that need no GPU: the library builds, loads, exports every symbol
include/fastged.h declares, and refuses to run without a CUDA device (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fastged.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fastged_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_00830_b200 import build, binding
    build.build()
    return binding.lib()


def test_header_declares_north_star_calls():
    names = _declared()
    for n in ("fastged_create", "fastged_solve_pair", "fastged_solve_batch", "fastged_destroy"):
        assert n in names


def test_exports_every_declared_symbol(lib):
    from paper_2605_00830_b200 import binding
    declared = _declared()
    assert set(declared) == set(binding.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_version(lib):
    from paper_2605_00830_b200 import binding
    assert "sm_100a" in binding.version()


def test_struct_layouts():
    from paper_2605_00830_b200 import binding
    assert C.sizeof(binding.GraphT) == 32
    assert C.sizeof(binding.CostsT) == 24
    assert C.sizeof(binding.ResultT) == 40


def test_no_device_fails_loudly(lib):
    """Without a GPU the library must refuse (FASTGED_ERR_CUDA), never compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2605_00830_b200 import binding
    with pytest.raises(binding.FastGedError) as e:
        binding.Handle(0)
    assert e.value.code == binding.ERR_CUDA


def test_built_for_sm100a(lib):
    import subprocess
    from paper_2605_00830_b200 import binding
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", binding.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_flag_constants_match_header():
    """The binding's flag values are the header's (FASTGED_FLAG_*; the approximate top-K shift in bits 8..11)."""
    from paper_2605_00830_b200 import binding
    src = open(os.path.join(ROOT, "include", "fastged.h")).read()
    vals = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define FASTGED_FLAG_([A-Z_]+) (\d+)u", src)}
    for name in ("TIMING", "DEBUG_WINDOW", "FORCE_LARGE", "VIRTUAL_SHARDS", "LAST_BY_TOTAL"):
        assert getattr(binding, "FLAG_" + name) == vals[name], name
    assert re.search(r"#define FASTGED_FLAG_APPROX\(shift\) \(\(uint32_t\)\(\(shift\) & 15\) << 8\)", src)
    assert [binding.FLAG_APPROX(s) for s in (0, 1, 15)] == [0, 256, 15 << 8]
    from oracle import oracle
    assert [oracle.APPROX(s) for s in (0, 1, 15)] == [0, 256, 15 << 8]
