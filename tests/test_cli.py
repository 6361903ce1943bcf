"""cli module: schedule dump (host only), bench protocol and
verify on the GPU."""

import json

import numpy as np
import pytest

from paper_2103_13577_b200 import cli


def _run(capsys, argv):
    rc = cli.main(argv)
    out = capsys.readouterr().out.strip().splitlines()[-1]
    return rc, json.loads(out)


def test_schedule_dump(capsys):
    rc, d = _run(capsys, ["schedule", "--nodes", "16", "--fanout", "1"])
    assert rc == 0 and d["num_rounds"] == 4 and d["message_count_paper"] == 64
    rc, d = _run(capsys, ["schedule", "--nodes", "16", "--fanout", "4"])
    assert d["num_rounds"] == 2 and d["message_count_paper"] == 128
    rc, d = _run(capsys, ["schedule", "--nodes", "9", "--fanout", "1"])
    assert [d["rounds"][-1][g] for g in range(8)] == [[8]] * 8


def test_root_sampling_protocol():
    a, short = cli.sample_roots(1000, 100, 7)
    b, _ = cli.sample_roots(1000, 100, 7)
    assert not short and np.array_equal(a, b) and len(set(a.tolist())) == 100
    c, short = cli.sample_roots(10, 100, 7)
    assert short and len(c) == 10


@pytest.mark.gpu
def test_bench_protocol(capsys, tmp_path):
    # acceptance 9: roots=100, trim=25 keeps 50; same roots across configs
    csvp = tmp_path / "runs.csv"
    rc, r1 = _run(capsys, ["bench", "--kronecker", "12", "8", "1", "--nodes", "4", "--fanout", "2",
                           "--roots", "100", "--trim", "25", "--csv", str(csvp)])
    assert rc == 0 and r1["roots_sampled"] == 100 and r1["roots_kept"] == 50
    assert abs(r1["teps_nominal"] * r1["mean_time"] - r1["num_edges"]) < 1e-3 * r1["num_edges"]
    rc, r2 = _run(capsys, ["bench", "--kronecker", "12", "8", "1", "--nodes", "4", "--fanout", "4",
                           "--roots", "100", "--trim", "25"])
    assert [x["root"] for x in r1["per_run"]] == [x["root"] for x in r2["per_run"]]
    assert [x["frontier_sizes"] for x in r1["per_run"]] == [x["frontier_sizes"] for x in r2["per_run"]]
    rc, r3 = _run(capsys, ["bench", "--kronecker", "12", "8", "1", "--nodes", "4",
                           "--strategy", "all2all", "--roots", "10", "--trim", "0"])
    assert rc == 0 and r3["roots_kept"] == 10
    assert csvp.read_text().splitlines()[0] == \
        "root,elapsed_s,levels,remote_messages,remote_vertices,buffer_high_water_max"


@pytest.mark.gpu
def test_verify_pass_and_negative_fixture(capsys, monkeypatch):
    rc, d = _run(capsys, ["verify", "--kronecker", "12", "8", "1", "--nodes", "9", "--fanout", "1",
                          "--roots", "5"])
    assert rc == 0 and d["ok"]
    # negative fixture: a corrupted engine result must be reported
    real = cli.engine.run

    def corrupted(g, p, root, cfg=None):
        d, st = real(g, p, root, cfg)
        if p.num_parts > 1:
            d.d = d.d.copy()
            d.d[np.flatnonzero(d.d != 0xFFFFFFFF)[-1]] += 1
        return d, st

    monkeypatch.setattr(cli.engine, "run", corrupted)
    rc, d = _run(capsys, ["verify", "--kronecker", "12", "8", "1", "--nodes", "2", "--fanout", "2",
                          "--roots", "2"])
    assert rc == 1 and not d["ok"] and d["got"] == d["expected"] + 1
