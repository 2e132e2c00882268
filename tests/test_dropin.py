"""Compiled drop-in proof: tests/dropin/dropin.c uses only the reference's
public header (pclab.h:1-93 -- its types, status codes and entry points)
and is linked against libpclab_b200.so. The CPU test compiles it against
the UNMODIFIED reference header where /root/reference is present (the build
container) and runs the host-only entry points; the GPU twin runs the
matrix / solve entry points through the same binary (or, on a box without
the reference, the same source compiled against include/pclab_b200.h, which
declares every pclab.h entry point with the same signature)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "dropin", "dropin.c")
LIBDIR = os.path.join(ROOT, "paper_2412_07127_b200")
OUT = os.path.join(ROOT, "build", "dropin")
REF_INC = "/root/reference/proj/include"


def build(inc: str, name: str) -> str:
    os.makedirs(OUT, exist_ok=True)
    exe = os.path.join(OUT, name)
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Werror", "-I", inc, SRC, "-L", LIBDIR, "-lpclab_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-lm", "-o", exe], check=True, capture_output=True, text=True)
    return exe


def test_dropin_host_entry_points_against_reference_header(tmp_path):
    if not os.path.exists(os.path.join(REF_INC, "pclab.h")):
        pytest.skip("reference header not present (build container only)")
    exe = build(REF_INC, "dropin_refhdr")
    r = subprocess.run([exe, "host"], cwd=tmp_path, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    assert "status_name 0 ok" in out and "status_name 3 numeric" in out and "status_name 5 internal" in out
    assert "param_count 997" in out
    assert "load_missing io" in out


@pytest.mark.gpu
def test_dropin_solves_through_the_reference_interface(tmp_path):
    exe = os.path.join(OUT, "dropin_refhdr")
    if not os.path.exists(exe):
        exe = build(os.path.join(ROOT, "tests", "dropin", "own"), "dropin_ownhdr")
    r = subprocess.run([exe, "gpu", str(tmp_path)], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    out = r.stdout
    for k in ("none", "jacobi", "ic0", "nic", "gnnic"):
        assert f"poisson3d {k} status ok" in out
    assert "duplicate format coo: entries not sorted or duplicate at (0, 1)" in out
