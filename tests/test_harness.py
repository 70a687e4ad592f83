"""The benchmark harness (paper_2212_08815_b200.harness) against the reference harness
(bench_cli.py): same flags, validation, CSV schemas and row order; on the GPU its
density outputs equal the reference harness's own (tests/golden/harness.npz)."""

import csv

import numpy as np
import pytest

from conftest import load_golden

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import harness as hz
from paper_2212_08815_b200 import network as nw


def test_config_validation_and_cli():
    with pytest.raises(ValueError, match="reps"):
        hz.BenchConfig(reps=2).validate()
    with pytest.raises(ValueError, match="densities"):
        hz.BenchConfig(densities=[0.0]).validate()
    with pytest.raises(ValueError, match="batch"):
        hz.BenchConfig(batches=[0]).validate()
    with pytest.raises(SystemExit) as e:
        hz.main(["bench", "--reps", "2"])
    assert e.value.code == 2
    args = hz.build_parser().parse_args(["bench", "--density", "1,50", "--batch", "1,4", "--full-scale"])
    cfg = hz.config_from_args(args)
    assert cfg.densities == [0.01, 0.5] and cfg.batches == [1, 4] and cfg.scale == 1.0 and cfg.input_hw == 224
    assert hz._twin_path("out/density.csv", "yolo_desk_nobn") == "out/density_yolo_desk_nobn.csv"
    with pytest.raises(ValueError, match="sparse_input"):
        hz.run_density_study(hz.BenchConfig(variant="sparse_filter"))


def test_csv_schema(tmp_path):
    rows = [hz.TimingRow("sparse_filter", 0.1, 1, 1, "strategy_i", r, 0.5 + r) for r in range(3)]
    p = tmp_path / "t.csv"
    hz.write_timing_csv(p, rows)
    got = list(csv.reader(open(p)))
    assert tuple(got[0]) == hz.TIMING_CSV_COLUMNS
    assert got[1] == ["sparse_filter", "0.1", "1", "1", "strategy_i", "0", "0.500000"]
    assert hz.summarize(rows) == [("sparse_filter", 0.1, 1, 1, "strategy_i", 1.5, 0.5)]
    d = tmp_path / "d.csv"
    hz.write_density_csv(d, [nw.DensityRecord(0.05, 3, "relu", 0.123456789)])
    assert list(csv.reader(open(d))) == [list(hz.DENSITY_CSV_COLUMNS), ["0.05", "3", "relu", "0.123457"]]


@pytest.mark.gpu
def test_harness_matches_reference_on_gpu(tmp_path):
    g = load_golden("harness.npz")
    fs.set_exact(True)  # bit-exact conv values -> identical densities for sparse_filter too
    try:
        for i in range(2):
            cfg = hz.BenchConfig(net_kind=str(g[f"b{i}__kind"]), scale=0.125, variant=str(g[f"b{i}__variant"]),
                                 densities=[0.1, 0.5], reps=3)
            timing, dens = hz.run_bench(cfg)
            keys = [f"{r.variant}|{r.density:g}|{r.batch}|{r.workers}|{r.strategy}|{r.rep}" for r in timing]
            assert keys == [str(k) for k in g[f"b{i}__timing_keys"]]
            assert all(r.seconds > 0 for r in timing)
            got = np.array([[r.input_density, r.layer_index, r.output_density] for r in dens])
            assert np.array_equal(got, g[f"b{i}__density"])
            assert [r.layer_kind for r in dens] == [str(k) for k in g[f"b{i}__density_kind"]]
    finally:
        fs.set_exact(False)
    cfg = hz.BenchConfig(net_kind="yolo_desk", scale=0.125, variant="sparse_input", densities=[0.2, 1.0], reps=3)
    for kind, rows in hz.run_density_study(cfg).items():
        assert np.array_equal(np.array([[r.input_density, r.layer_index, r.output_density] for r in rows]),
                              g[f"study_{kind}"]), kind
    # the CLI end to end
    t, d = tmp_path / "timing.csv", tmp_path / "density.csv"
    assert hz.main(["bench", "--scale", "0.125", "--density", "10", "--timing-csv", str(t),
                    "--density-csv", str(d)]) == 0
    assert len(list(csv.reader(open(t)))) == 1 + 2 * 3  # variant + dense baseline, 3 reps
