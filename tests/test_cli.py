"""CLI over the B200 backend: same verbs, formats and
exit codes as the reference CLI; printed documents byte-identical to the
reference's (goldens)."""

import json

import pytest

import golden_io as G
from paper_1801_08058_b200.cli import main
from paper_1801_08058_b200.serialize import print_function


def _write(tmp_path, name, doc):
    p = tmp_path / name
    p.write_text(json.dumps(doc, indent=2) + "\n")
    return p


def test_grad_documents_byte_identical_to_reference(tmp_path, capsys):
    for case in G.load("gradients.json.gz"):
        f = _write(tmp_path, "fn.gf.json", case["fn"])
        wrt = ",".join(f"p{case['fn']['parameters'].index(w)}" for w in case["wrt"])
        assert main(["grad", str(f), "--wrt", wrt]) == 0
        got = capsys.readouterr().out
        assert got == json.dumps(case["grad_fn"], indent=2) + "\n", case["name"]


def test_printer_round_trips_reference_documents():
    for case in G.load("corpus.json.gz")[:50]:
        text = json.dumps(case["fn"], indent=2) + "\n"
        assert print_function(G.fn_of(case["fn"])) == text


def test_validate_and_exit_codes(tmp_path, capsys):
    f = _write(tmp_path, "ok.gf.json", G.load("corpus.json.gz")[0]["fn"])
    assert main(["validate", str(f)]) == 0
    bad = dict(G.load("corpus.json.gz")[0]["fn"])
    bad = json.loads(json.dumps(bad))
    bad["results"] = [[999, 0]]
    b = _write(tmp_path, "bad.gf.json", bad)
    assert main(["validate", str(b)]) == 2
    assert main(["validate", str(tmp_path / "missing.gf.json")]) == 4
    assert main(["nope"]) == 4
    (tmp_path / "junk.gf.json").write_text("{not json")
    assert main(["validate", str(tmp_path / "junk.gf.json")]) == 2


def test_plan_matches_reference_listing_arena(tmp_path, capsys):
    case = G.load("corpus.json.gz")[3]
    f = _write(tmp_path, "fn.gf.json", case["fn"])
    assert main(["plan", str(f)]) == 0
    out = capsys.readouterr().out
    assert out.strip().splitlines()[-1].startswith("arena ")


@pytest.mark.gpu
def test_run_matches_reference_outputs(tmp_path, capsys):
    case = G.load("corpus.json.gz")[5]
    f = _write(tmp_path, "fn.gf.json", case["fn"])
    args = ["run", str(f), "--out", str(tmp_path / "out")]
    for i, d in enumerate(case["inputs"]):
        args += ["--input", str(_write(tmp_path, f"in{i}.tensor.json", d))]
    assert main(args) == 0
    for j, want in enumerate(case["outputs_opt"]):
        got = json.loads((tmp_path / "out" / f"result{j}.tensor.json").read_text())
        assert G.max_abs_diff(G.logical(got), G.logical(want)) <= (1e-12 if want["element_type"] == "F64" else 1e-6)
