"""CPU-side checks of the boundary: libhmg.so loads and exports every symbol
include/hmg.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "hmg.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^HMG_API [^(]*?\b(hmg_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("hmg_build_hierarchy", "hmg_apply_helmholtz", "hmg_vcycle", "hmg_fgmres_solve"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2511_16808_b200 import build
    lib = ctypes.CDLL(build.build())
    for n in declared():
        assert hasattr(lib, n), n


def test_binding_covers_every_declared_symbol():
    from paper_2511_16808_b200 import hmg
    assert sorted(hmg.EXPORTED) == declared()
    assert hmg.launch_count() == 0
    assert "sm_100a" in hmg.version()


def test_library_has_sm100a_code_only():
    import subprocess
    from paper_2511_16808_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
