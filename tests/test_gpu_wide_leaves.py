"""GPU: the wide-leaf pre-tests (per-triangle containment slabs, per-leaf
oriented boxes) are result-neutral on adversarial dense meshes.

A large search ball (maxDistanceFraction x sqrt(F) >= 27) makes the bake build
leaves of up to 15 triangles with their TPlane / LPlane records. The dense
mesh gets exact duplicate faces (ties: the lower face index must win),
degenerate faces (a repeated vertex), zero-area collinear faces, slivers a
1e-9 hair off an edge, a shuffled face order and, in one case, a far
translation (the pre-tests' slack scales with the coordinates' magnitude).
Hit faces must equal the CPU port's bit for bit."""
import numpy as np
import pytest

from paper_2605_26137_b200 import fixtures as fx
from paper_2605_26137_b200.mesh import TriangleMesh

from test_gpu_configs import check_pair

pytestmark = pytest.mark.gpu


def adversarial_pair(frac, offset, seed):
    p = fx.bake_pair(40, 8, 256, frac=frac, seed=seed, name="wide")
    V, F = p.dense.positions, p.dense.faces
    rng = np.random.default_rng(seed)
    k = 400
    dup = F[rng.choice(len(F), k, replace=False)]
    deg = np.stack([F[:k, 0], F[:k, 0], F[:k, 1]], 1)
    idx = rng.choice(len(F), k, replace=False)
    mids = 0.5 * (V[F[idx, 0]] + V[F[idx, 1]])
    mid_ids = len(V) + np.arange(k)
    col = np.stack([F[idx, 0], F[idx, 1], mid_ids], 1)
    hair = mids + 1e-9 * rng.standard_normal((k, 3))
    hair_ids = len(V) + k + np.arange(k)
    sliver = np.stack([F[idx, 0], hair_ids, F[idx, 1]], 1)
    faces = np.concatenate([F, dup, deg, col, sliver])
    faces = faces[rng.permutation(len(faces))]
    shift = np.asarray(offset, dtype=np.float64)
    dense = TriangleMesh(np.concatenate([V, mids, hair]) + shift, faces)
    lo = p.lowpoly
    low = TriangleMesh(lo.positions + shift, lo.faces, uvs=lo.uvs, face_uvs=lo.face_uvs)
    return fx.BakePair("wide", dense, low, p.res, frac)


@pytest.mark.parametrize("frac,offset,seed", [
    (0.3, (0.0, 0.0, 0.0), 11),     # leaf cap 8
    (0.5, (0.0, 0.0, 0.0), 12),     # leaf cap 14
    (0.5, (3000.0, -1500.0, 700.0), 13),  # far from the origin: slack ~ 2^-16 of 3000
])
def test_wide_leaf_pretests_are_result_neutral(gpu_ctx, port, frac, offset, seed):
    p = adversarial_pair(frac, offset, seed)
    scale = frac * np.sqrt(p.dense.face_count())
    assert scale >= 27.0  # wide leaves: the planes are built
    out, o = check_pair(p, port)
    assert (o["face"] >= 0).sum() > 10_000
