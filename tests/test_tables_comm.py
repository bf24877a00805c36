"""Host-side mirrors: MDLB bundle I/O (tables.py:20-77) and the analytic
volume model (comm.py:67-157), against reference-made fixtures and the
reference tests' known answers."""

import numpy as np
import pytest

from golden_util import GOLDEN, toy_bundle_path
from paper_2503_04398_b200 import comm, tables


@pytest.mark.parametrize("ci", range(3))
def test_bundle_roundtrip_byte_identical(ci, tmp_path):
    src = toy_bundle_path(ci)
    b = tables.read_bundle(src)
    assert b.token_table.n_clusters == 2 and len(b.expert_labels) == 8
    tables.write_bundle(tmp_path / "copy.bin", b)
    assert (tmp_path / "copy.bin").read_bytes() == src.read_bytes()


def test_bundle_rejects_bad_input(tmp_path):
    (tmp_path / "bad.bin").write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(tables.TableError):
        tables.read_bundle(tmp_path / "bad.bin")
    with pytest.raises(tables.TableError):
        tables.read_bundle(GOLDEN / "toy.npz")
    blob = toy_bundle_path(0).read_bytes()
    (tmp_path / "short.bin").write_bytes(blob[:-3])
    with pytest.raises(tables.TableError):
        tables.read_bundle(tmp_path / "short.bin")


def test_bundle_lookup_tables_bit_identical_to_reference_dtypes():
    b = tables.read_bundle(toy_bundle_path(1))
    assert b.ngram_table.probs.dtype == np.float64 and b.ngram_table.counts.dtype == np.int64
    assert b.ngram_table.best.dtype == np.int16 and b.ngram_table.confidence.dtype == np.float32


def closed_dense(G, B, S, k):
    return 3 * B * S * (G - 1) / G + 2 * B * S * k * (G - 1) / G ** 2


def closed_sharded(G, B, S, k, a):
    return B * S * (G - 1) / G + 2 * B * S * k * (1 - a) / G


def test_volume_closed_forms_and_points():
    # test_comm.py:32-50, test_acceptance.py:33-47
    for G in (2, 4, 8, 16):
        for k in (1, 2, 6):
            d = comm.pipeline_volume(comm.dense_pipeline(G, 3.0, 7.0, k))
            assert abs(d.total - closed_dense(G, 3.0, 7.0, k)) <= 1e-12
            for a in np.linspace(0, 1, 11):
                s = comm.pipeline_volume(comm.sharded_pipeline(G, 3.0, 7.0, k, float(a)))
                assert abs(s.total - closed_sharded(G, 3.0, 7.0, k, a)) <= 1e-12
    assert comm.pipeline_volume(comm.dense_pipeline(8, 1, 1, 1)).total == pytest.approx(2.84375)
    assert comm.pipeline_volume(comm.sharded_pipeline(8, 1, 1, 6, 1.0)).total == pytest.approx(0.875)
    tp = comm.pipeline_volume(comm.tensor_parallel_pipeline(8))
    lo = comm.saving_ratio(tp, comm.pipeline_volume(comm.sharded_pipeline(8, k=6, alpha=0.0)))
    hi = comm.saving_ratio(tp, comm.pipeline_volume(comm.sharded_pipeline(8, k=6, alpha=1.0)))
    assert lo == pytest.approx(0.3214285714, abs=1e-9) and hi == pytest.approx(0.75, abs=1e-9)
    with pytest.raises(comm.CommError):
        comm.volume_collective("all_to_all", 4, 1, 1, alpha=1.5)
    with pytest.raises(comm.CommError):
        comm.volume_collective("ring_exchange", 4, 1, 1)


def test_sweep_alpha_affine():
    rows = comm.sweep_alpha(8, 6, 11)
    diffs = np.diff([r["sharded_volume"] for r in rows])
    assert np.allclose(diffs / 0.1, -2 * 6 / 8, atol=1e-9)
    with pytest.raises(comm.CommError):
        comm.sweep_alpha(8, 6, 1)


def test_predicted_saving_table():
    """BASELINE.md §3 predictions (model and +SAG)."""
    def saving(G, k, a, sag):
        d = comm.pipeline_volume(comm.dense_pipeline(G, 1, 1, k))
        spec = comm.sharded_pipeline_with_sag if sag else comm.sharded_pipeline
        return comm.saving_ratio(d, comm.pipeline_volume(spec(G, 1, 1, k, a)))
    assert saving(8, 2, 0.5, False) == pytest.approx(0.633, abs=1e-3)
    assert saving(8, 2, 0.5, True) == pytest.approx(0.347, abs=1e-3)
    assert saving(8, 6, 0.9, False) == pytest.approx(0.740, abs=1e-3)
    assert saving(8, 6, 0.9, True) == pytest.approx(0.517, abs=1e-3)
