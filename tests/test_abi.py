"""CPU: the C-ABI library loads and exports every symbol include/asv.h declares
(no compute calls — there is no GPU here)."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "asv.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(asv_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("asv_decode_attention", "asv_attn_plan_build", "asv_engine_run", "asv_run_config_jsonl",
                 "asv_dfs_batch", "asv_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(h, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) <= bound, set(declared_symbols()) - bound


def test_struct_mirrors_match_the_library():
    """Every ctypes mirror has the size of the C struct the library was compiled with."""
    import ctypes as C
    from paper_2605_23389_b200 import _lib
    h = _lib.lib()
    for cname, mirror in (("asv_attn_shape", _lib.AttnShape), ("asv_attn_plan", _lib.AttnPlan),
                          ("asv_attn_args", _lib.AttnArgs), ("asv_linear_args", _lib.LinearArgs),
                          ("asv_engine_opts", _lib.EngineOpts), ("asv_engine_stats", _lib.EngineStats)):
        assert h.asv_struct_size(cname.encode()) == C.sizeof(mirror), cname
    assert h.asv_struct_size(b"nope") == -1


def test_library_is_built_for_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_2605_23389_b200", "libasv.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_error_mapping_matches_reference_exceptions():
    from paper_2605_23389_b200 import engine
    with pytest.raises(RuntimeError, match="config missing workload"):
        engine.run_config_jsonl({"policy": "aligned"})
    with pytest.raises(RuntimeError, match="unknown policy"):
        engine.run_config_jsonl({"workload": {"count": 1}, "policy": "nope"})


def test_header_is_c_and_links(tmp_path):
    """include/asv.h is a C header: a C translation unit compiles against it, links against
    libasv.so and runs the GPU-free entry points (what a cgo / JNI / N-API shim does)."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or "/opt/gcc/bin/gcc"
    exe = tmp_path / "abi_smoke"
    pkg = os.path.join(ROOT, "paper_2605_23389_b200")
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-L", pkg, "-lasv",
                        f"-Wl,-rpath,{pkg}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and r.stdout.startswith("ok 8388608"), (r.returncode, r.stdout, r.stderr)
