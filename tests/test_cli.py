"""CLI (reference cli.py): file formats and exit codes on CPU; `run`/`grad` on the GPU."""

import json

import numpy as np
import pytest

from oracle import layersim_oracle as orc
from paper_2506_04891_b200 import cli


def _circuit_doc(n=4):
    return {"n": n, "layers": [
        {"gate": "ry", "pattern": "all", "role": "encoding"},
        {"gate": "rx", "pattern": "all", "role": "trainable"},
        {"gate": "cnot", "pattern": "ring"},
        {"gate": "rzz", "pattern": "explicit", "wires": [[0, 1], [2, 3]], "role": "fixed",
         "values": [[0.3], [-0.7]]},
    ]}


def _files(tmp_path, batch=3):
    c = tmp_path / "c.json"
    c.write_text(json.dumps(_circuit_doc()))
    rng = np.random.default_rng(3)
    p = tmp_path / "p.json"
    p.write_text(json.dumps({"trainable": rng.uniform(-3, 3, 4).tolist(),
                             "encoding": rng.uniform(0, 3, (batch, 4)).tolist()}))
    return c, p


def test_parse_circuit_roundtrip(tmp_path):
    c, p = _files(tmp_path)
    circ = cli.load_circuit(c)
    assert circ.n == 4 and len(circ.layers) == 4
    assert circ.trainable_count == 4 and circ.encoding_count == 4
    tr, en = cli.load_params(p)
    assert tr.shape == (4,) and en.shape == (3, 4)


@pytest.mark.parametrize("doc,code", [
    ({"layers": []}, 2),                                                  # no n
    ({"n": 2, "layers": [{"gate": "nope", "pattern": "all"}]}, 2),         # unknown gate
    ({"n": 2, "layers": [{"gate": "rx", "pattern": "all"}]}, 2),           # missing role
])
def test_bad_circuit_exit_codes(tmp_path, doc, code):
    c = tmp_path / "bad.json"
    c.write_text(json.dumps(doc))
    assert cli.main(["run", "--circuit", str(c)]) == code


def test_missing_file_exit_code(tmp_path):
    assert cli.main(["run", "--circuit", str(tmp_path / "none.json")]) == 2


@pytest.mark.gpu
def test_cli_run_and_grad_match_oracle(tmp_path, capsys):
    c, p = _files(tmp_path)
    circ = cli.load_circuit(c)
    tr, en = cli.load_params(p)
    assert cli.main(["run", "--circuit", str(c), "--params", str(p)]) == 0
    vals = np.array([float(x) for x in capsys.readouterr().out.split()])
    ref = orc.gradient(circ, tr, en, batch=3)
    np.testing.assert_allclose(vals, ref["value"], atol=1e-5)
    assert cli.main(["grad", "--circuit", str(c), "--params", str(p)]) == 0
    out = json.loads(capsys.readouterr().out)
    np.testing.assert_allclose(out["value"], ref["value"], atol=1e-5)
    np.testing.assert_allclose(out["grads"], ref["grads"], atol=1e-4)


def test_bench_families_and_qubit_parser():
    """The harness's circuit families and argument parsing (reference bench.py:81-136,
    cli.py:30-38), checked on CPU against the oracle through the emulator."""
    from emulator import Emulator
    from paper_2506_04891_b200 import harness
    from paper_2506_04891_b200.schedule import compile_circuit

    assert cli._parse_qubits("4..6") == (4, 5, 6) and cli._parse_qubits("4,8") == (4, 8)
    with pytest.raises(ValueError):
        cli._parse_qubits("6..4")
    with pytest.raises(ValueError):
        harness.BenchConfig("nope", (4,), (1,))
    for fam in harness.FAMILIES:
        c = harness.build_circuit(fam, 5, 2)
        tr, en = harness.draw_params(c, 3, 0, 5)
        res = Emulator(compile_circuit(c, M=4, R=2)).gradient(tr, en, 3, None)
        ref = orc.gradient(c, tr, en, batch=3)
        np.testing.assert_allclose(res["grads"], ref["grads"], atol=1e-9)


@pytest.mark.gpu
def test_bench_subcommand_writes_reports(tmp_path):
    pytest.importorskip("torch").cuda.is_available() or pytest.skip("needs a GPU")
    out = tmp_path / "r.csv"
    rc = cli.main(["bench", "--family", "ibm", "--qubits", "6,8", "--batch", "4", "--blocks", "2",
                   "--reps", "2", "--warmup", "1", "--objective", "forward+backward", "--out", str(out)])
    assert rc == 0
    import csv

    rows = list(csv.reader(open(out)))
    assert tuple(rows[0])[:10] == ("family", "n", "batch", "phase", "plan_source", "mean_s", "std_s", "reps",
                                   "warmup", "seed")
    assert len(rows) == 1 + 2 * 3 and {r[3] for r in rows[1:]} == {"forward", "backward", "total"}
    cross = list(csv.reader(open(tmp_path / "r_crossover.csv")))
    assert cross[0] == ["family", "n", "batch", "gate", "pattern", "role", "kernel"] and len(cross) > 1
