"""Tensor file format (interp.py:34-70) and the `run` document
(cli.py:155-188) around the B200 executor."""

import json

import numpy as np
import pytest

from conftest import GOLDEN


def _gemm_inputs(d):
    from paper_2107_00555_b200.tensorio import TensorValue

    d.mkdir()
    # the reference's own CLI fixture (pkg/tests/test_cli.py:14-23)
    TensorValue.of(np.array([[1.0, 2.0], [3.0, 4.0]])).save(d / "A.json")
    TensorValue.of(np.eye(2)).save(d / "B.json")
    TensorValue.of(np.zeros((2, 2))).save(d / "C.json")
    TensorValue.of(np.array(1.0)).save(d / "alpha.json")
    TensorValue.of(np.array(0.0)).save(d / "beta.json")
    return d


def test_tensor_value_format_and_round_trip(tmp_path):
    from paper_2107_00555_b200.tensorio import TensorValue

    t = TensorValue.of(np.array([[1.5, -2.0], [3.0, 4.25]]))
    assert t.to_json() == {"dtype": "f64", "shape": [2, 2], "data": [1.5, -2.0, 3.0, 4.25]}
    # 0-d values come out with shape [1], as the reference's (np.ascontiguousarray)
    assert TensorValue.of(np.array(7)).to_json() == {"dtype": "i64", "shape": [1], "data": [7]}
    assert TensorValue.of(np.array([True, False])).dtype == "bool"
    assert TensorValue.of(np.arange(3), "i32").array.dtype == np.int32
    p = tmp_path / "t.json"
    t.save(p)
    assert p.read_text().endswith("\n")
    back = TensorValue.load(p)
    assert back.dtype == "f64" and np.array_equal(back.array, t.array)
    assert json.loads(p.read_text())["shape"] == [2, 2]
    with pytest.raises(ValueError):
        TensorValue.from_json({"dtype": "f16", "shape": [], "data": [0]})


def test_run_document_missing_input_is_code_1(tmp_path):
    from paper_2107_00555_b200.tensorio import RunError, run_document

    d = tmp_path / "in"
    d.mkdir()
    with pytest.raises(RunError) as ex:
        run_document(GOLDEN / "graphs" / "gemm.raw.json", {"NI": 2, "NJ": 2, "NK": 2}, d)
    assert ex.value.code == 1 and "missing input tensor" in str(ex.value)


@pytest.mark.gpu
def test_run_document_identity_product(tmp_path):
    """pkg/tests/test_cli.py:43-50 through the B200 executor."""
    from paper_2107_00555_b200.tensorio import run_document

    d = _gemm_inputs(tmp_path / "in")
    doc = run_document(GOLDEN / "graphs" / "gemm.raw.json", {"NI": 2, "NJ": 2, "NK": 2}, d)
    assert doc["outputs"]["C"]["data"] == [1.0, 2.0, 3.0, 4.0]
    assert doc["outputs"]["C"]["shape"] == [2, 2]
    assert doc["report"]["per_rank"][0]["map_iterations"] >= 8
