"""Regenerates tests/golden/*.npz from the REFERENCE's own translation units
(oracle/_ref/libmfref.so, built by oracle/Makefile from /root/reference).

Run here (the container that has /root/reference):
    python tests/golden/make_golden.py
The .npz files are committed; the GPU box never reads /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings  # noqa: E402
from paper_2605_26137_b200 import fixtures as fx  # noqa: E402

# Small cases whose outputs pin the oracle and the CUDA path.
BAKE_CASES = {
    # name: (n_dense, n_low, res, frac, seed, low_scale)
    "tiny": (24, 4, 64, 0.01, 7, 1.0),
    "small": (48, 8, 128, 0.01, 11, 1.0),
    "cage": (48, 8, 128, 0.05, 5, 1.04),
}


def bake_case(ref, name):
    nd, nl, res, frac, seed, scale = BAKE_CASES[name]
    p = fx.bake_pair(nd, nl, res, frac, seed, scale, name=name)
    g = ref.raster_gbuffer(p.lowpoly, res)
    out = ref.bake(p.lowpoly, p.dense, res, p.bbox_diagonal, frac, 4, debug=True)
    return dict(
        res=res, frac=frac, diag=p.bbox_diagonal, seed=seed, n_dense=nd, n_low=nl, low_scale=scale,
        valid=g.valid, reliable=g.reliable, position=g.position, normal=g.normal, tangent=g.tangent,
        bitangent=g.bitangent, rgb=out["rgb"], rgb_raw=out["rgb_raw"], face=out["face"], ts=out["ts"],
        n_node=out["n_node"], n_tri=out["n_tri"])


def spatial_case(ref):
    sphere = ref.fixture(0, 2, r=0.5)  # icosphere(2)
    q = ref.random_points(300, (-1, -1, -1), (1, 1, 1), 41)
    f, ds, pt, bary = ref.closest_within(sphere, q)
    fb, dsb, ptb, baryb = ref.closest_within(sphere, q, 0.2)
    uvs = ref.fixture(1, 24, 24, r=0.5)  # uvSphere(24, 24)
    o = ref.random_points(300, (-1.5, -1.5, -1.5), (1.5, 1.5, 1.5), 21)
    tgt = ref.random_points(300, (-0.4, -0.4, -0.4), (0.4, 0.4, 0.4), 23)
    d = ref.random_units(300, 22)
    d[::2] = (tgt - o)[::2] / np.linalg.norm((tgt - o)[::2], axis=1, keepdims=True)
    rf, rt, ru, rv = ref.raycast_first(uvs, o, d)
    return dict(ico_pos=sphere.positions, ico_faces=sphere.faces, q=q, cp_face=f, cp_dist=ds, cp_point=pt,
                cp_bary=bary, cpw_face=fb, cpw_dist=dsb, uvs_pos=uvs.positions, uvs_faces=uvs.faces,
                ray_o=o, ray_d=d, ray_face=rf, ray_t=rt, ray_u=ru, ray_v=rv)


def tangent_case(ref):
    m = ref.fixture(0, 1, r=0.5)
    m = fx.assign_cell_uvs(m, 10)
    frames = ref.wedge_tangents(m)
    vn = ref.vertex_normals(ref.fixture(0, 3, r=0.5))
    return dict(pos=m.positions, faces=m.faces, uvs=m.uvs, face_uvs=m.face_uvs, frames=frames,
                vn_mesh_pos=ref.fixture(0, 3, r=0.5).positions, vn_mesh_faces=ref.fixture(0, 3, r=0.5).faces,
                vnormals=vn)


def kat_case(ref):
    """Small known-answer inputs of proj/tests/test_bake.cpp run through the reference."""
    from paper_2605_26137_b200.mesh import TriangleMesh
    out = {}
    # off-density face (test_bake.cpp:145-169)
    m = TriangleMesh([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0], [1, 0, 200]], [[0, 1, 2], [0, 2, 3], [1, 4, 2]],
                     uvs=[[0.05, 0.05], [0.35, 0.05], [0.35, 0.35], [0.05, 0.35], [0.65, 0.05]],
                     face_uvs=[[0, 1, 2], [0, 2, 3], [1, 4, 2]])
    g = ref.raster_gbuffer(m, 128)
    out.update(od_valid=g.valid, od_reliable=g.reliable, od_rgb=ref.transfer_normals(g, m, m.bbox_diagonal()))
    # distance filter (test_bake.cpp:185-200)
    q = fx.identity_quad()
    far = fx.identity_quad()
    far.positions[:, 2] += 0.08
    g = ref.raster_gbuffer(q, 32)
    out.update(far_valid=g.valid, far_rgb=ref.transfer_normals(g, far, float(np.sqrt(2.0))))
    # fill rule (test_bake.cpp:135-143) and one triangle covering the atlas (:77-96)
    out["fill_valid"] = ref.raster_gbuffer(q, 8).valid
    tri = TriangleMesh([[0, 0, 0], [2, 0, 0], [0, 2, 0]], [[0, 1, 2]], uvs=[[0, 0], [2, 0], [0, 2]],
                       face_uvs=[[0, 1, 2]])
    g = ref.raster_gbuffer(tri, 32)
    out.update(tri_valid=g.valid, tri_position=g.position, tri_normal=g.normal, tri_tangent=g.tangent)
    # lone texel chebyshev ball (test_bake.cpp:253-274)
    valid = np.zeros(121, np.uint8)
    valid[5 * 11 + 5] = 1
    img = np.zeros((121, 3), np.uint8)
    img[5 * 11 + 5] = (10, 20, 30)
    out["lone_valid"] = valid
    out["lone_in"] = img
    out["lone_out"] = ref.dilate_seams(img, 11, 11, 3, 11, valid, 2)
    return out


# markSurfaceBand cases (signfield/sign_grid.cpp:23-69): (fixture args, res, bandVoxels, dilateRadius, domain)
BAND_CASES = {
    "ico4": ((0, 4, 0, 0, 0.5), 64, 1.0, 2, None),
    "plane": ((4, 8, 8, 0, 0.5), 48, 1.0, 2, None),
    "torus": ((5, 24, 12, 0, 0.5), 40, 1.5, 1, None),
    "domain": ((0, 3, 0, 0, 0.4), 32, 1.0, 2, (-0.6, -0.6, -0.6, 0.6, 0.6, 0.6)),
}


def band_case(ref):
    out = {}
    for name, (fa, res, band, dil, dom) in BAND_CASES.items():
        m = ref.fixture(*fa)
        labels, dist, grid = ref.surface_band(m, res, band, dil, dom)
        out.update({f"{name}_pos": m.positions, f"{name}_faces": m.faces, f"{name}_labels": labels,
                    f"{name}_dist": dist, f"{name}_grid": grid,
                    f"{name}_params": np.array([res, band, dil], np.float64),
                    f"{name}_domain": np.array(dom if dom else [np.nan] * 6, np.float64)})
    return out


def concat(a, b):
    from paper_2605_26137_b200.mesh import TriangleMesh
    return TriangleMesh(np.vstack([a.positions, b.positions]),
                        np.vstack([a.faces, b.faces + a.vertex_count()]).astype(np.int32))


def views_case(ref):
    """renderView / castVisibility (render/raster.cpp:12-102, visibility.cpp:13-59)
    through the reference: nested spheres (sealed inner shell: zero hits), a
    duplicated mesh (depth ties keep the lower face) and a star blob."""
    nested = concat(ref.fixture(0, 3, r=0.5), ref.fixture(0, 2, r=0.2))
    blob = ref.fixture(2, 24, 32, 11, 0.5)
    dup = concat(ref.fixture(0, 1, r=0.5), ref.fixture(0, 1, r=0.5))
    cams = ref.fibonacci_cameras(8, 0.55, 96)
    out = dict(cams=cams)
    for name, m in (("nested", nested), ("blob", blob), ("dup", dup)):
        vn = ref.vertex_normals(m)
        face, depth, pos, nrm = ref.render_views(m, cams, 96, vn)
        out.update({f"{name}_pos_in": m.positions, f"{name}_faces": m.faces, f"{name}_vn": vn,
                    f"{name}_face": face, f"{name}_depth": depth, f"{name}_hits": ref.cast_visibility(m, 32, 96)})
        if name == "blob":  # position / normal images of two views; RasterOptions::backfaceCull
            out.update(blob_position=pos[:2], blob_normal=nrm[:2])
            # reversed winding: culling drops the near shell, the far one shows
            from paper_2605_26137_b200.mesh import TriangleMesh
            rev = TriangleMesh(m.positions, np.ascontiguousarray(m.faces[:, ::-1]))
            cf, cd, _, _ = ref.render_views(rev, cams[:2], 96, vn, cull=True)
            out.update(blob_cull_face=cf, blob_cull_depth=cd)
    return out


def texfuse_case(ref):
    """texfuse over a small G-buffer (fuse.cpp:66-280, mips.cpp:96-112): three
    standard views of a dense blob, synthetic colours; the reference's edge
    masks, mip chains, partial atlases, incidence maps and blend."""
    p = fx.bake_pair(24, 4, 64, name="texfuse")
    g = ref.raster_gbuffer(p.lowpoly, 64)
    cams = ref.standard_cameras(0.8)[[0, 4, 8]]
    vres = 96
    face, depth, pos, _ = ref.render_views(p.dense, cams, vres)
    col = (0.5 + 0.5 * np.sin(np.concatenate([5.0 * pos[..., :1], 3.0 * pos[..., 1:2] + 1.0,
                                              7.0 * pos[..., 2:3]], -1))) * (face >= 0)[..., None]
    col = col.astype(np.float32)
    diag = p.bbox_diagonal
    masks, chains, parts, samps, incs = [], [], [], [], []
    for i in range(3):
        m = ref.edge_mask(pos[i], face[i], diag, 0.02)
        chain, nm = ref.build_mips(col[i], 6, 0.2)
        c, sp = ref.backproject_view(g.position, g.valid, 64, cams[i], vres, 3, nm, chain, m)
        inc = ref.incidence_map(g.position, g.normal, g.valid, 64, cams[i], vres, depth[i], diag, 0.005)
        masks.append(m)
        chains.append(chain)
        parts.append(c)
        samps.append(sp)
        incs.append(inc)
    priors = np.array([1.0, 1.0, 0.3])
    out, filled = ref.blend_views(np.stack(parts), np.stack(samps), np.stack(incs), priors)
    return dict(g_position=g.position, g_normal=g.normal, g_valid=g.valid, cams=cams, vres=vres, diag=diag,
                v_face=face, v_depth=depth, v_pos=pos, colors=col, masks=np.stack(masks), chains=np.stack(chains),
                parts=np.stack(parts), sampled=np.stack(samps), incidence=np.stack(incs), priors=priors,
                blend=out, filled=filled)


def main():
    ref = bindings.ref()
    if sys.argv[1:] == ["texfuse"]:  # regenerate only this file
        np.savez_compressed(os.path.join(HERE, "texfuse.npz"), **texfuse_case(ref))
        return
    np.savez_compressed(os.path.join(HERE, "texfuse.npz"), **texfuse_case(ref))
    np.savez_compressed(os.path.join(HERE, "views.npz"), **views_case(ref))
    np.savez_compressed(os.path.join(HERE, "band.npz"), **band_case(ref))
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **kat_case(ref))
    for name in BAKE_CASES:
        np.savez_compressed(os.path.join(HERE, f"bake_{name}.npz"), **bake_case(ref, name))
    np.savez_compressed(os.path.join(HERE, "spatial.npz"), **spatial_case(ref))
    np.savez_compressed(os.path.join(HERE, "tangents.npz"), **tangent_case(ref))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
