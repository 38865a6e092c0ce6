"""CPU: the C-ABI libraries load and export every declared entry point (no
compute calls - there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mfbake.h")
LIB = os.path.join(ROOT, "paper_2605_26137_b200", "libmfbake.so")
CPPLIB = os.path.join(ROOT, "paper_2605_26137_b200", "libmeshforge_b200.so")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mf_[a-z0-9_]+)\s*\(", text)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_header_declares_the_boundary():
    names = declared()
    for must in ("mf_raster_gbuffer", "mf_transfer_normals", "mf_dilate_seams", "mf_bake_normal_map",
                 "mf_bake_normal_map_dev", "mf_bvh_build", "mf_bvh_closest_within", "mf_bvh_raycast_first",
                 "mf_wedge_tangents", "mf_vertex_normals", "mf_closest_point_brute", "mf_raycast_first_brute"):
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "libmfbake.so not built (run __graft_entry__.build())"
    missing = [n for n in declared() if n not in exported(LIB)]
    assert not missing, missing


def test_python_bindings_cover_the_header():
    from paper_2605_26137_b200 import capi
    bound = {n for n, _, _ in capi.SIGNATURES}
    assert set(declared()) <= bound
    lib = capi.load()
    assert lib.mf_abi_version() == 1
    assert b"sm_100a" in lib.mf_version()


def test_context_creation_fails_cleanly_without_a_device():
    from paper_2605_26137_b200 import capi
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("a device is present")
    with pytest.raises(capi.MeshforgeError) as e:
        capi.Context(0)
    assert e.value.status == -4  # MF_ERR_NO_DEVICE: no silent CPU path


def test_cpp_api_library_exports_the_reference_api():
    assert os.path.exists(CPPLIB)
    out = subprocess.run(["nm", "-DC", "--defined-only", CPPLIB], capture_output=True, text=True, check=True).stdout
    for sig in ("meshforge::rasterizeGBuffer(", "meshforge::transferNormals(", "meshforge::dilateSeams(",
                "meshforge::Bvh::Bvh(", "meshforge::Bvh::closestPointWithin(", "meshforge::Bvh::raycastFirst(",
                "meshforge::computeWedgeTangents(", "meshforge::computeVertexNormals(",
                "meshforge::closestPointBrute(", "meshforge::raycastFirstBrute("):
        assert sig in out, sig
