"""The command line front end (paper_2503_10017_b200/cli.py) against the
reference CLI contract (tools/fastnn_cli.cpp, docs/formats.md): files written
by ``gen``, the JSON-lines / report / bench schemas of ``match`` and
``bench``, ``verify`` against the exhaustive mutual-NN oracle, exit codes."""
import json
import os

import numpy as np
import pytest

from paper_2503_10017_b200 import cli

REPORT_FIELDS = ("backend,metric,precision,height1,width1,height2,width2,dim,k,grid_stride,max_iters,"
                 "convergence_fraction,block_size,seed,subsample_us,forward_nn_us,reverse_nn_us,harvest_us,"
                 "a_block_fetches,b_block_fetches,iterations,samples,converged,converged_fraction,half_saturated,"
                 "half_saturation_events,hybrid_full_argmin_agreement,matches_emitted,duplicates_dropped")


def test_gen_writes_pair_truth_manifest(tmp_path):
    import paper_2503_10017_b200 as fnl
    out = tmp_path / "pair"
    assert cli.main(["gen", "--height", "16", "--width", "12", "--dim", "8", "--seed", "5", "-o", str(out)]) == 0
    d1, d2 = fnl.read_fmap(str(out / "d1.fmap")), fnl.read_fmap(str(out / "d2.fmap"))
    assert d1.shape == d2.shape == (16, 12, 8)
    truth = json.loads((out / "truth.json").read_text())
    assert list(truth)[:5] == ["height", "width", "dim", "noise_sigma", "permute"]
    assert sorted(truth["map"]) == list(range(16 * 12))  # a full permutation
    p = fnl.gen_matched_pair(16, 12, 8, 5, 0.0, "random")
    assert np.array_equal(d1, p["d1"]) and np.array_equal(truth["map"], p["truth"])
    man = json.loads((out / "manifest.json").read_text())
    assert man == {"fmap1": "d1.fmap", "fmap2": "d2.fmap", "ground_truth": "truth.json"}


@pytest.mark.parametrize("argv", [
    ["match", "-o", "x.jsonl"],                                   # no inputs
    ["match", "a.fmap", "b.fmap", "-o", "x.jsonl", "--convergence", "1.5"],
    ["match", "a.fmap", "b.fmap", "-o", "x.jsonl", "--backend", "quantum"],
    ["bench", "--sizes", "512"],
    ["bench", "--backends", "single,warp"],
    ["gen", "--height", "0", "-o", "d"],
    ["verify", "a.fmap", "b.fmap"],                               # --matches missing
])
def test_usage_errors_exit_2(argv, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    with pytest.raises(SystemExit) as e:
        raise SystemExit(cli.main(argv))
    assert e.value.code == 2


def test_match_missing_file_exits_1(tmp_path):
    assert cli.main(["match", str(tmp_path / "a.fmap"), str(tmp_path / "b.fmap"), "-o", str(tmp_path / "m.jsonl")]) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["single", "tensor"])
def test_gen_match_verify_roundtrip(tmp_path, backend, capsys):
    import paper_2503_10017_b200 as fnl
    out = tmp_path / "pair"
    assert cli.main(["gen", "--height", "32", "--width", "24", "--seed", "7", "--noise", "0.05", "-o", str(out)]) == 0
    mpath, rpath = tmp_path / "m.jsonl", tmp_path / "r.csv"
    rc = cli.main(["match", "--manifest", str(out / "manifest.json"), "--backend", backend, "--metric", "dot",
                   "--stride", "4", "--seed", "42", "-o", str(mpath), "--report", str(rpath),
                   "--report-format", "csv"])
    assert rc == 0
    lines = mpath.read_text().splitlines()
    got = np.array([[json.loads(x)[k] for k in ("i", "j", "iter")] for x in lines], dtype=np.uint32).reshape(-1, 3)
    want, _ = fnl.reciprocal_match(fnl.read_fmap(str(out / "d1.fmap")), fnl.read_fmap(str(out / "d2.fmap")),
                                   backend=backend, metric="dot", stride=4)
    assert np.array_equal(got, want)
    assert all(x.startswith('{"i":') for x in lines)
    header, row = rpath.read_text().splitlines()
    assert header.replace(" ", "") == REPORT_FIELDS
    assert row.split(",")[REPORT_FIELDS.split(",").index("seed")] == "42"
    capsys.readouterr()
    assert cli.main(["verify", "--matches", str(mpath), "--manifest", str(out / "manifest.json"),
                     "--metric", "dot"]) == 0
    assert "violations: 0" in capsys.readouterr().out
    # a corrupted match file fails verification with exit code 1
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"i":0,"j":1,"iter":1}\n{"i":0,"j":2,"iter":1}\n')
    assert cli.main(["verify", "--matches", str(bad), "--manifest", str(out / "manifest.json"),
                     "--metric", "dot"]) == 1


@pytest.mark.gpu
def test_bench_csv_schema(tmp_path):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--sizes", "32x24,16x12", "--block-sizes", "256", "--backends",
                     "double,single,hybrid,tensor", "--metric", "dot", "--repeats", "2", "-o", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == cli.BENCH_HEADER
    rows = [x.split(",") for x in lines[1:]]
    assert len(rows) == 8 and [r[5] for r in rows[:4]] == ["double", "single", "hybrid", "tensor"]
    for r in rows:
        assert float(r[9]) > 0 and int(r[12]) > 0 or r[5] == "tensor"
        assert (r[14] != "") == (r[5] in ("hybrid", "tensor"))
    # the double loop's fetch law: b = ceil(P/BS)^2 (nn.cpp:103)
    P = 32 * 24
    assert int(rows[0][13]) == (-(-P // 256)) ** 2
    js = tmp_path / "b.json"
    assert cli.main(["bench", "--sizes", "16x12", "--backends", "single", "--repeats", "1", "--format", "json",
                     "-o", str(js)]) == 0
    assert list(json.loads(js.read_text())[0]) == cli.BENCH_HEADER.split(",")
