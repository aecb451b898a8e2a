"""TrialRecord CSV (trial.hpp:16-148 schema + measured columns) and the
sweep driver's resume / canonical-merge contract (sweep.hpp:195-289), on CPU."""
import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))

from paper_2308_16877_b200 import trial as T  # noqa: E402


def test_header_keeps_reference_columns_first():
    ref = T.REF_HEADER.split(",")
    assert len(ref) == 22 and T.HEADER.split(",")[:22] == ref
    assert T.HEADER.split(",") == list(T.TrialRecord.__dataclass_fields__)


def test_record_round_trip_and_shortest_doubles():
    r = T.TrialRecord("blackscholes", "taf", "memo(out:5:1:0.5) out(price[i])", "warp", 4096, 64, 32, 16,
                      1 << 22, 42, 0, "OK", "", "mape", 0.1 + 0.2, 0.125, 0.0, 0.108, 0.104, 1.04, 0, 0,
                      4.0e10, 1.04, "lattice=1024")
    row = T.to_csv_row(r)
    assert "0.30000000000000004" in row  # repr round trip (fmtnum.hpp:13-19)
    assert '"memo(out:5:1:0.5) out(price[i])"' not in row or "," in r.directive
    back = T.from_csv_row(row)
    assert back == r


def test_failed_record_and_quoting():
    r = T.TrialRecord("kmeans", "perfo", 'perfo(ini:10) in(pt[i:32]) out(dist[i:64])', status="FAILED",
                      reason='ConfigError: trip count, "quoted"')
    back = T.from_csv_row(T.to_csv_row(r))
    assert back.reason == r.reason and back.status == "FAILED"


def test_sort_key_orders_configuration_fields():
    a = T.TrialRecord("binomial", "iact", "x", num_teams=1)
    b = T.TrialRecord("binomial", "iact", "x", num_teams=2)
    c = T.TrialRecord("blackscholes", "taf", "a")
    assert sorted([c, b, a], key=lambda r: r.sort_key()) == [a, b, c]


def test_sweep_points_parse_and_are_unique():
    import sweep
    from paper_2308_16877_b200 import engine as E
    pts = sweep.points(["blackscholes", "binomial", "kmeans", "lavamd"])
    keys = [sweep.point_key(*p) for p in pts]
    assert len(set(keys)) == len(keys)
    for _, _, d in pts:
        E.parse_directive(d)  # every directive is valid reference grammar
    assert {p[0] for p in pts} == {"blackscholes", "binomial", "kmeans", "lavamd"}


def test_sweep_merge_resume_contract(tmp_path):
    import sweep
    out = tmp_path / "s.csv"
    recs = [T.TrialRecord("lavamd", "taf", f"d{i}", trial=i) for i in (3, 1, 2)]
    # two ranks' parts, one duplicated point (a resumed run re-wrote it)
    p0 = Path(f"{out}.part.0")
    p1 = Path(f"{out}.part.1")
    p0.write_text("".join(f"k{r.trial}\t{T.to_csv_row(r)}\n" for r in recs[:2]))
    p1.write_text(f"k{recs[2].trial}\t{T.to_csv_row(recs[2])}\n" + f"k{recs[0].trial}\t{T.to_csv_row(recs[0])}\n")
    assert set(sweep.load_done(p0)) == {"k3", "k1"}
    merged = sweep.merge(out, [p0, p1], {"points": 3})
    lines = out.read_text().splitlines()
    assert lines[0] == T.HEADER and len(lines) == 4
    assert [r.directive for r in merged] == ["d1", "d2", "d3"]  # canonical order
    assert not p0.exists() and not p1.exists()
    assert json.loads(out.with_suffix(".csv.json").read_text())["points"] == 3


@pytest.mark.gpu
def test_run_trial_small_points():
    from paper_2308_16877_b200 import engine as E
    w = T.make_workload("blackscholes", 64 * 64 * 16, 16)
    r = T.run_trial(w, f"memo(out:5:1:0.5) {T.SECTIONS['blackscholes']}")
    assert r.status == "OK" and r.technique == "taf" and abs(r.approx_rate - 0.125) < 1e-12
    assert r.baseline_cost > 0 and r.approx_cost > 0 and r.error_metric == "mape"
    bad = T.run_trial(w, f"perfo(ini:10) {T.SECTIONS['blackscholes']} level(warp)")
    assert bad.status in ("OK", "FAILED")
    k = T.make_workload("kmeans", 64 * 64 * 4, 4, separation=30.0, max_iters=5)
    rk = T.run_trial(k, f"perfo(random:25) {T.SECTIONS['kmeans']} level(warp)")
    assert rk.status == "OK" and rk.error_metric == "mcr" and rk.baseline_iters >= 1
    lv = T.make_workload("lavamd", 0, 1, boxes1d=4, particles=128)
    rl = T.run_trial(lv, f"memo(out:2:2:0.1) {T.SECTIONS['lavamd']} level(team)")
    assert rl.status == "OK" and rl.n == 64
