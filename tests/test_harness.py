"""The experiment harness (paper_1808_10481_b200/harness.py):
catalog and configuration errors on CPU; on the GPU the paper's studies
through the device stepper must reproduce the reference's goldens and rate
bands (test_stepper1d.cpp:323-371, SPEC.md acceptance 1-6, 9)
and the CSV files must follow emit_csv's format."""
import csv
import math
import os

import pytest

from paper_1808_10481_b200 import harness as HR


def test_list_and_configuration_errors(capsys):
    assert HR.cli_main(["list"]) == 0
    out = capsys.readouterr().out
    assert len([ln for ln in out.splitlines() if ln.strip()]) == 7
    assert HR.cli_main(["run", "no-such-experiment"]) == 1
    assert HR.cli_main(["run", "standing-wave-1d", "--resolutions", ""]) == 1       # empty resolution list
    assert HR.cli_main(["run", "standing-wave-1d", "--resolutions", "20,10"]) == 1  # not increasing
    assert HR.cli_main(["run", "acoustics-2d", "--variant", "modified"]) == 1
    assert HR.cli_main(["dispersion"]) == 1


def test_rate_fit_is_the_reference_rule():
    hs = [0.2, 0.1, 0.05, 0.025]
    es = [1e-3 * (h / 0.2) ** 6 for h in hs]
    r, used = HR.convergence_rate(hs, es)
    assert abs(r - 6.0) < 1e-12 and used == 4
    r, used = HR.convergence_rate(hs, [1e-3, 1e-20, 1e-20, 1e-20])  # below the 100 eps floor
    assert r is None and used == 1


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(f))


@pytest.mark.gpu
def test_standing_wave_table1(tmp_path):
    # test_stepper1d.cpp:323-338 goldens (2 %) and SPEC acceptance 1 (6.00 +- 0.3)
    assert HR.cli_main(["run", "standing-wave-1d", "--m", "2", "--cfl", "0.9", "--out", str(tmp_path)]) == 0
    errs = rows(tmp_path / "errors.csv")
    gold = {10: 1.5081e-04, 20: 2.3521e-06, 40: 3.6708e-08, 80: 5.7460e-10}
    for r in errs:
        assert float(r["l2_error"]) == pytest.approx(gold[int(r["K"])], rel=0.02)
    rate = rows(tmp_path / "rates.csv")
    assert len(rate) == 1 and abs(float(rate[0]["rate"]) - 6.00) < 0.3
    assert list(errs[0].keys()) == ["experiment", "variant", "m", "cfl", "K", "h", "field", "l2_error", "steps",
                                    "wall_seconds"]


@pytest.mark.gpu
def test_variable_speed_table2(tmp_path):
    # forced variable speed (test_stepper1d.cpp:340-355): goldens and 6.02 +- 0.3
    assert HR.cli_main(["run", "variable-speed-1d", "--m", "2", "--out", str(tmp_path)]) == 0
    gold = {10: 5.3628e-06, 20: 8.0000e-08, 40: 1.2426e-09, 80: 1.9781e-11}
    for r in rows(tmp_path / "errors.csv"):
        assert float(r["l2_error"]) == pytest.approx(gold[int(r["K"])], rel=0.02)
    assert abs(float(rows(tmp_path / "rates.csv")[0]["rate"]) - 6.02) < 0.3


@pytest.mark.gpu
def test_modified_advection_table3(tmp_path):
    # single-field modified scheme (test_stepper1d.cpp:357-371): goldens, 5.98 +- 0.4
    assert HR.cli_main(["run", "advection-modified-1d", "--m", "2", "--out", str(tmp_path)]) == 0
    gold = {10: 1.298e-03, 20: 2.212e-05, 40: 3.541e-07}
    for r in rows(tmp_path / "errors.csv"):
        assert float(r["l2_error"]) == pytest.approx(gold[int(r["K"])], rel=0.02)
    assert abs(float(rows(tmp_path / "rates.csv")[0]["rate"]) - 5.98) < 0.4


@pytest.mark.gpu
def test_dual_hermite_and_pv_modified(tmp_path):
    # Dual-Hermite m = 2 (test_stepper1d.cpp:373-387 goldens); modified P-V m = 2 (SPEC acceptance 4: 5.93 +- 0.4)
    assert HR.cli_main(["run", "standing-wave-1d", "--m", "2", "--variant", "dual-hermite",
                        "--out", str(tmp_path / "dh")]) == 0
    gold = {10: 5.4033e-04, 20: 2.0392e-05, 40: 6.8730e-07, 80: 2.2202e-08}
    for r in rows(tmp_path / "dh" / "errors.csv"):
        assert float(r["l2_error"]) == pytest.approx(gold[int(r["K"])], rel=0.02)
    assert HR.cli_main(["run", "pv-modified-1d", "--m", "2", "--out", str(tmp_path / "pv")]) == 0
    assert abs(float(rows(tmp_path / "pv" / "rates.csv")[0]["rate"]) - 5.93) < 0.4


@pytest.mark.gpu
@pytest.mark.parametrize("m,rate", [(0, 1.86), (1, 1.88), (2, 6.01), (3, 6.74)])
def test_2d_acoustics_rates_spec_band(tmp_path, m, rate):
    # SPEC acceptance 5: 2D acoustics rates at CFL 0.9 within +-0.4 of
    # (1.86, 1.88, 6.01, 6.74) for m = 0..3, device Gauss L2 (l2_error_2d)
    assert HR.cli_main(["run", "acoustics-2d", "--m", str(m), "--out", str(tmp_path / "a")]) == 0
    got = float(rows(tmp_path / "a" / "rates.csv")[0]["rate"])
    assert abs(got - rate) < 0.4, (m, got, rate)


@pytest.mark.gpu
def test_2d_acoustics_maxwell_and_pulse(tmp_path):
    # SPEC acceptance 9 (Maxwell m = 4, CFL 0.8: >= 4 orders) and the pulse
    assert HR.cli_main(["run", "maxwell-tm-2d", "--m", "4", "--cfl", "0.8", "--out", str(tmp_path / "mx")]) == 0
    es = [float(r["l2_error"]) for r in rows(tmp_path / "mx" / "errors.csv")]
    assert es == sorted(es, reverse=True) and es[0] / es[-1] >= 1e4
    assert HR.cli_main(["run", "gaussian-reflect-2d", "--m", "3", "--out", str(tmp_path / "g")]) == 0
    g = rows(tmp_path / "g" / "errors.csv")
    assert math.isfinite(float(g[0]["l2_error"])) and float(g[0]["l2_error"]) <= 2.0


@pytest.mark.gpu
@pytest.mark.parametrize("m", [0, 1, 2, 3])
@pytest.mark.parametrize("cfl", [0.1, 0.5, 0.9])
def test_conservation_trace(tmp_path, m, cfl):
    # SPEC acceptance 6: Q^h / R^h within 1e-10 over 100 steps
    assert HR.conserve(m, cfl, 100, out=str(tmp_path)) < 1e-10
    assert os.path.exists(tmp_path / "conservation.csv")
