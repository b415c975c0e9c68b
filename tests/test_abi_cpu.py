"""The C ABI library without a GPU: it loads, exports every symbol that
include/systec.h declares, and the host-side argument checks answer before any
CUDA call.  No compute calls here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "systec.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"SYSTEC_API\s+[\w\s\*]*?\b(systec_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2406_09266_b200 import load
    return load()


def test_header_declares_the_north_star_call():
    syms = header_symbols()
    assert "systec_mttkrp" in syms and "systec_plan_execute" in syms and len(syms) >= 12


def test_library_exports_every_header_symbol(lib):
    from paper_2406_09266_b200 import EXPORTS
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert set(header_symbols()) == set(EXPORTS)


def test_status_strings_and_version(lib):
    assert lib.systec_status_string(0) == b"ok"
    assert lib.systec_status_string(3) == b"index outside [0, dim)"
    assert lib.systec_version() == 100
    assert lib.systec_last_bad_entry() == -1


def test_host_argument_checks_need_no_gpu(lib):
    vp = ctypes.c_void_p
    # order outside 2..5 -> UNSUPPORTED, before any CUDA call
    assert lib.systec_mttkrp(7, 10, 0, None, None, vp(16), 4, vp(4096), None) == 2
    assert lib.systec_mttkrp(1, 10, 0, None, None, vp(16), 4, vp(4096), None) == 2
    # dim < 1, nnz < 0 -> ARG
    assert lib.systec_mttkrp(3, 0, 0, None, None, vp(16), 4, vp(4096), None) == 1
    assert lib.systec_mttkrp(3, 10, -1, None, None, vp(16), 4, vp(4096), None) == 1
    # dim or nnz beyond int32 -> UNSUPPORTED (a sort key wider than 64 bits is supported: wide plans)
    assert lib.systec_mttkrp(5, 1 << 31, 0, None, None, vp(16), 4, vp(1 << 30), None) == 2
    assert lib.systec_mttkrp(5, 10, (1 << 31) - 64, vp(16), vp(16), vp(16), 4, vp(1 << 30), None) == 2
    # null idx with nnz > 0 -> ARG
    assert lib.systec_mttkrp(3, 10, 5, None, None, vp(16), 4, vp(4096), None) == 1
    # R < 1 -> ARG
    assert lib.systec_mttkrp(3, 10, 0, None, None, vp(16), 0, vp(4096), None) == 1
    # C overlapping B -> ALIAS
    assert lib.systec_mttkrp(3, 10, 0, None, None, vp(4096), 4, vp(4096 + 16), None) == 4
    # plan-less calls
    assert lib.systec_plan_execute(None, vp(16), 4, vp(4096), None) == 1
    assert lib.systec_plan_stats(None, None) == 1
    out = ctypes.c_void_p()
    assert lib.systec_plan_create(ctypes.byref(out), 6, 10, 0, None, None, None) == 2
    assert not out.value
    # the testing pass entry: bad form / dim / null -> -ARG, misaligned -> -UNSUPPORTED
    assert lib.systec_testing_cpd_pass(2, 10, vp(16), vp(16), vp(16), vp(16), 1, None) == -1
    assert lib.systec_testing_cpd_pass(0, 0, vp(16), vp(16), vp(16), vp(16), 1, None) == -1
    assert lib.systec_testing_cpd_pass(1, 10, None, vp(16), vp(16), vp(16), 1, None) == -1
    assert lib.systec_testing_cpd_pass(1, 10, vp(20), vp(16), vp(16), vp(16), 1, None) == -2


def test_product_path_has_no_oracle_dependency():
    """The CUDA path never imports, links or calls oracle/ (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2406_09266_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    text = f.read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), fn
                assert "mttkrp_oracle" not in text and "liboracle" not in text, fn
    for fn in os.listdir(os.path.join(ROOT, "oracle")):
        if fn.endswith((".py", ".c")):
            with open(os.path.join(ROOT, "oracle", fn)) as f:
                text = f.read()
            assert not re.search(r"^\s*(import|from)\s+paper_2406_09266_b200", text, re.M), fn
            assert "libsystec" not in text and '#include "systec.h"' not in text, fn


def test_sass_shows_bulk_async_copies_and_vector_reductions(lib):
    """The sm_100a kernel c2 runs (fixed-rank R = 32 build) really uses the TMA engine (UBLKCP) for the stream,
    16-byte gathers and vector fp32 reductions (checked in the cubin, no GPU)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_2406_09266_b200 import LIB_PATH
    sass = subprocess.run(["cuobjdump", "-sass", "-fun",
                           "_ZN6systec17mttkrp_sym_kernelILi3ELi8ELi1ELi4ELb0ELb0ELb0ELi0ELi32EEEvNS_7KParamsE", LIB_PATH],
                          capture_output=True, text=True).stdout
    elfs = subprocess.run(["cuobjdump", "-lelf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elfs
    assert "UBLKCP" in sass
    assert "REDG.E.ADD.F32x4" in sass
    assert "LDG.E.128" in sass
    assert "SYNCS" in sass          # mbarrier waits


def test_header_is_plain_c_and_example_builds(lib):
    """include/systec.h is valid C11 and a plain C program links against the
    library (run on the GPU box by tests/test_gpu_parity.py)."""
    import shutil
    import subprocess
    import tempfile
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    out = os.path.join(tempfile.mkdtemp(), "mttkrp_c")
    subprocess.check_call(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "mttkrp_c.c"), "-o", out,
                           "-L", os.path.join(ROOT, "paper_2406_09266_b200"), "-lsystec",
                           "-L", "/usr/local/cuda/lib64", "-lcudart",
                           "-Wl,-rpath," + os.path.join(ROOT, "paper_2406_09266_b200")])
    assert os.path.exists(out)


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The binding's ctypes mirrors of systec_stats / systec_exec_opts / systec_plan_opts have the
    C layout (sizes and field offsets compiled from include/systec.h)."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    from paper_2406_09266_b200.systec import SystecExecOpts, SystecPlanOpts, SystecStats
    src = tmp_path / "layout.c"
    fields = [("systec_stats", n) for n, _ in SystecStats._fields_] + \
             [("systec_exec_opts", n) for n, _ in SystecExecOpts._fields_] + \
             [("systec_plan_opts", n) for n, _ in SystecPlanOpts._fields_]
    body = "\n".join(f'    printf("%s %s %zu\\n", "{t}", "{f}", offsetof({t}, {f}));' for t, f in fields)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "systec.h"\nint main(void) {\n'
                   '    printf("size systec_stats %zu\\n", sizeof(systec_stats));\n'
                   '    printf("size systec_exec_opts %zu\\n", sizeof(systec_exec_opts));\n'
                   '    printf("size systec_plan_opts %zu\\n", sizeof(systec_plan_opts));\n' + body + "\n    return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
    got = {(a, b): int(c) for a, b, c in (l.split() for l in out if l)}
    assert got[("size", "systec_stats")] == ctypes.sizeof(SystecStats)
    assert got[("size", "systec_exec_opts")] == ctypes.sizeof(SystecExecOpts)
    assert got[("size", "systec_plan_opts")] == ctypes.sizeof(SystecPlanOpts)
    for t, cls in (("systec_stats", SystecStats), ("systec_exec_opts", SystecExecOpts),
                   ("systec_plan_opts", SystecPlanOpts)):
        for f, _ in cls._fields_:
            assert got[(t, f)] == getattr(cls, f).offset, (t, f)


def test_host_call_rejects_wrong_torch_dtypes_and_shapes(lib):
    """Torch host tensors are passed to systec_mttkrp_host in place, so a
    wrong dtype or shape must raise before the call."""
    import torch

    import paper_2406_09266_b200 as systec
    idx = torch.zeros((5, 3), dtype=torch.int32)
    vals = torch.zeros(5, dtype=torch.float32)
    B = torch.zeros((10, 4), dtype=torch.float32)
    with pytest.raises(TypeError):
        systec.mttkrp_host(3, 10, idx.long(), vals, B)
    with pytest.raises(TypeError):
        systec.mttkrp_host(3, 10, idx, vals.double(), B)
    with pytest.raises(TypeError):
        systec.mttkrp_host(3, 10, idx, vals, B.double())
    with pytest.raises(TypeError):
        systec.mttkrp_host(3, 10, idx[:, :2].contiguous(), vals, B)
    with pytest.raises(TypeError):
        systec.mttkrp_host(3, 10, idx, vals, B, C=torch.zeros((10, 5)))
