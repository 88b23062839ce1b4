"""C-ABI library: builds, loads without a GPU, exports every symbol that
include/lfoam.h declares, and the binding declares exactly those (-m "not gpu")."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "lfoam.h")


def header_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^LF_API\s+[\w\s\*]*?\b(\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2507_18268_b200 import build
    return build.build()


def test_header_parses():
    names = header_functions()
    for required in ["mesh_create", "field_set", "laplacian_assemble", "ldu_amul", "pcg_solve",
                     "laplacianFoam_step"]:
        assert required in names


def test_library_exports_every_header_symbol(libpath):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libpath], text=True)
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    # nothing else leaks (hidden visibility for internals)
    extra = [n for n in exported if n.startswith("lf") and n not in header_functions()]
    assert not extra, extra


def test_binding_matches_header(libpath):
    import paper_2507_18268_b200 as P
    assert sorted(P.SIGNATURES) == header_functions()
    L = P.lib()  # loads on a CPU-only box (CUDA runtime is linked statically)
    assert L.lf_version() == 2
    assert L.lf_status_string(1) == b"LF_ERR_INVALID_ARG"


def test_binding_struct_layouts(tmp_path):
    """ctypes structs have the C layout of include/lfoam.h (gcc sizeof/offsetof)."""
    import ctypes as C

    import paper_2507_18268_b200 as P
    from paper_2507_18268_b200 import lfoam as B
    checks = {"lf_solver_controls": (B.Controls, ["preconditioner", "reserved"]),
              "lf_laplacian_params": (B.Params, ["variable_DT"]),
              "lf_mesh_desc": (B.MeshDesc, ["renumber", "c"]),
              "lf_patch_desc": (B.PatchDesc, ["neighb_rank", "sf"]),
              "lf_solver_perf": (B.Perf, ["n_iterations", "reserved"])}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "lfoam.h"', "int main(void){"]
    for name, (_, fields) in checks.items():
        src.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f in fields:
            src.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    src.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = dict(ln.split() for ln in subprocess.check_output([str(exe)], text=True).splitlines())
    for name, (cls, fields) in checks.items():
        assert int(got[name]) == C.sizeof(cls), name
        for f in fields:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, (name, f)


def test_kernels_built_for_sm100a(libpath):
    out = subprocess.check_output(["cuobjdump", "--list-elf", libpath], text=True)
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", libpath], text=True)
    assert "k_phase1" in sass and "k_assemble" in sass


def test_no_device_without_gpu(libpath):
    """On a CPU-only box the context call fails with a status, not a crash."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2507_18268_b200 as P
    with pytest.raises(P.LfoamError) as e:
        P.Context(0)
    assert e.value.status in (1, 4)


def test_product_does_not_import_oracle():
    """The product path never references oracle/ (independence rule)."""
    pkg = os.path.join(ROOT, "paper_2507_18268_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "lfoam_oracle" not in txt, f


def test_binding_option_ids_match_header():
    """lfoam.py's option names map to the lf_option values include/lfoam.h
    declares (LF_OPT_<NAME> = id), one for one."""
    import paper_2507_18268_b200.lfoam as L
    src = open(HEADER).read()
    body = re.search(r"typedef enum \{([^}]*)\} lf_option;", src).group(1)
    ids = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"LF_OPT_(\w+)\s*=\s*(\d+)", body)}
    alias = {"solve_variant": "variant"}
    assert {alias.get(k, k): v for k, v in ids.items()} == L.OPTIONS
