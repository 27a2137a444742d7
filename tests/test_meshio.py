"""ASCII mesh interchange with the reference (mesh.py:175-200): the oracle/GPU runs and the
reference exchange geometry through this format.  The fixtures were written by the
unmodified reference's write_mesh (tools/make_golden_meshfile.py)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN


def _meshes():
    from paper_1506_05957_b200 import make_icosphere
    from paper_1506_05957_b200.configs import _rbc_pair
    from paper_1506_05957_b200.meshes import Mesh

    pair = _rbc_pair()
    return {"ico2_ref.mesh": make_icosphere(2),
            "rbc2_ref.mesh": Mesh(pair.vertices, pair.triangles,
                                  np.repeat(np.arange(2), pair.n_panels // 2))}


@pytest.mark.parametrize("name", ["ico2_ref.mesh", "rbc2_ref.mesh"])
def test_write_mesh_is_byte_identical_to_the_reference(name, tmp_path):
    from paper_1506_05957_b200 import write_mesh

    mesh = _meshes()[name]
    out = tmp_path / name
    write_mesh(out, mesh)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


@pytest.mark.parametrize("name", ["ico2_ref.mesh", "rbc2_ref.mesh"])
def test_read_mesh_reads_the_reference_files_exactly(name, tmp_path):
    from paper_1506_05957_b200 import read_mesh, write_mesh

    mesh = _meshes()[name]
    back = read_mesh(os.path.join(GOLDEN, name))
    assert np.array_equal(back.vertices, mesh.vertices)  # %.17g round-trips doubles exactly
    assert np.array_equal(back.triangles, mesh.triangles)
    assert np.array_equal(back.tags, mesh.tags)
    write_mesh(tmp_path / "again.mesh", back)
    again = read_mesh(tmp_path / "again.mesh")
    assert np.array_equal(again.vertices, back.vertices) and np.array_equal(again.tags, back.tags)


def test_read_mesh_rejects_bad_headers(tmp_path):
    from paper_1506_05957_b200 import read_mesh

    bad = tmp_path / "bad.mesh"
    bad.write_text("3 1\n0 0 0\n1 0 0\n0 1 0\n0 1 2 0\n0 1 2 0\n")
    read_mesh(bad)  # extra trailing rows are ignored like the reference (max_rows)
    bad.write_text("4 1\n0 0 0\n1 0 0\n0 1 0\n")
    with pytest.raises(ValueError):
        read_mesh(bad)
