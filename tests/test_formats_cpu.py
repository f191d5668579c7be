"""File formats: NRTF and weights JSON are byte-compatible with
the reference (linalg.py:72-117, operators.py:325-378) -- files written by either side
read back identically on the other."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


def _ref():
    if not os.path.isdir(REF):
        pytest.skip("reference not present (build container only)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from streamgnn import linalg, models, operators

    return linalg, models, operators


def test_nrtf_roundtrip_and_errors(tmp_path):
    from paper_2603_20622_b200 import ConfigError, read_tensor, write_tensor

    for dt in (np.float32, np.float64):
        a = np.arange(12, dtype=dt).reshape(3, 4) / 7
        p = str(tmp_path / f"t_{np.dtype(dt).name}.nrtf")
        write_tensor(p, a)
        b = read_tensor(p)
        assert b.dtype == dt and np.array_equal(a, b)
    with pytest.raises(ConfigError):
        write_tensor(str(tmp_path / "x.nrtf"), np.zeros(3))
    bad = tmp_path / "bad.nrtf"
    bad.write_bytes(b"XXXX" + b"\0" * 30)
    with pytest.raises(ConfigError):
        read_tensor(str(bad))


def test_nrtf_compatible_with_reference(tmp_path):
    linalg, _, _ = _ref()
    from paper_2603_20622_b200 import read_tensor, write_tensor

    a = np.random.default_rng(0).standard_normal((5, 3))
    p1, p2 = str(tmp_path / "ours.nrtf"), str(tmp_path / "ref.nrtf")
    write_tensor(p1, a)
    linalg.write_tensor(p2, a)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    assert np.array_equal(linalg.read_tensor(p1), read_tensor(p2))


def test_weights_json_compatible_with_reference(tmp_path):
    _, models, operators = _ref()
    from paper_2603_20622_b200 import load_weights, make_bundle, save_weights

    for model, dims in (("gcn", [4, 5, 3]), ("gin", [3, 3]), ("gat", [4, 6])):
        ref = models.make_bundle(model, dims)
        ours = make_bundle(model, dims)
        p1, p2 = str(tmp_path / f"{model}_ours.json"), str(tmp_path / f"{model}_ref.json")
        save_weights(ours, p1)
        operators.save_weights(ref, p2)
        a, b = load_weights(p2), operators.load_weights(p1)
        assert a["model"] == b["model"] == model
        for la, lb in zip(a["layers"], b["layers"]):
            assert (la.in_dim, la.out_dim) == (lb.in_dim, lb.out_dim)
            for k in la.tensors:
                assert np.array_equal(la.tensors[k], lb.tensors[k])
