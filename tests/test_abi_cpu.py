"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/mc.h declares, its struct layouts match the ctypes mirror, and calls
fail cleanly (no crash) when no device is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mc.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:mc_status|int64_t|int32_t|const char\*)\s+(mc_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2209_01158_b200 import build
    build.build()
    from paper_2209_01158_b200 import mc
    return mc.load()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["mc_create", "mc_set_continuum", "mc_set_coupling", "mc_step_decoupled",
                 "mc_step_coupled", "mc_run", "mc_destroy", "mc_get_state", "mc_error_string",
                 "mc_nlmc_build", "mc_nlmc_get", "mc_nlmc_basis"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2209_01158_b200 import mc
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in mc.EXPORTS
    out = subprocess.run(["nm", "-D", "--defined-only", mc.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mc_\w+)$", out, re.M))
    assert set(_declared()) <= exported
    assert lib.mc_abi_version() == 2


def test_struct_layouts_match_header(tmp_path):
    from paper_2209_01158_b200 import mc
    prog = tmp_path / "layout.c"
    fields = {
        "mc_options": [f[0] for f in mc.mc_options._fields_],
        "mc_continuum_desc": [f[0] for f in mc.mc_continuum_desc._fields_],
        "mc_coupling_desc": [f[0] for f in mc.mc_coupling_desc._fields_],
        "mc_step_report": [f[0] for f in mc.mc_step_report._fields_],
        "mc_nlmc_desc": [f[0] for f in mc.mc_nlmc_desc._fields_],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void){"]
    for s, fs in fields.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f in fs:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    prog.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c99", "-o", str(exe), str(prog)], check=True)
    got = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for s, fs in fields.items():
        cls = getattr(mc, s)
        assert int(got[s]) == C.sizeof(cls), s
        for f in fs:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def test_create_without_device_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2209_01158_b200 import mc
    ctx = C.c_void_p()
    opt = mc.mc_options(tau=0.1, rtol=1e-12)
    st = lib.mc_create(C.byref(ctx), 2, C.byref(opt))
    assert st == mc.MC_ERR_CUDA
    assert b"device" in lib.mc_error_string(None)
    assert not ctx.value


def test_argument_validation_before_device(lib):
    from paper_2209_01158_b200 import mc
    ctx = C.c_void_p()
    assert lib.mc_create(C.byref(ctx), 0, C.byref(mc.mc_options(tau=0.1))) == mc.MC_ERR_ARG
    assert lib.mc_create(C.byref(ctx), 2, C.byref(mc.mc_options(tau=-1.0))) == mc.MC_ERR_ARG
    assert lib.mc_create(C.byref(ctx), 2, C.byref(mc.mc_options(tau=0.1, rtol=2.0))) == mc.MC_ERR_ARG
    assert lib.mc_create(C.byref(ctx), 2, None) == mc.MC_ERR_ARG
    assert lib.mc_destroy(None) == mc.MC_OK


def test_product_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_2209_01158_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
