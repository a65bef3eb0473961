"""The run/verify CLI (python -m paper_1410_1726_b200 run), modelled on the
reference's test_cli.py:14-64 verify flow.  CPU: the CLI's wide-precision
checker against the oracle, argument errors.  GPU: end-to-end runs whose
CSV rows must verify."""

import csv

import numpy as np
import pytest

from oracle import naive
from paper_1410_1726_b200 import cli


class TestChecker:
    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("trans", "ntc")
    def test_gemv_checker_matches_oracle(self, tag, trans):
        rng = np.random.default_rng(5)
        m, n = 70, 2100
        a = naive.fill(rng, (m, n), tag)
        xl, yl = (n, m) if trans == "n" else (m, n)
        x, y = naive.fill(rng, xl, tag), naive.fill(rng, yl, tag)
        want, bound = cli.check_gemv(trans, 0.7, a, x, -0.3, y, np.finfo(naive.DTYPES[tag]).eps, panel=512)
        ref = naive.naive_gemv(trans, 0.7, a, x, -0.3, y)
        assert np.max(np.abs(want - ref)) <= bound
        assert bound > 0

    @pytest.mark.parametrize("tag", "sdcz")
    @pytest.mark.parametrize("uplo", "lu")
    def test_symv_checker_matches_oracle(self, tag, uplo):
        rng = np.random.default_rng(6)
        d = 1300
        vals = naive.fill(rng, (d, d), tag)
        herm = tag in "cz"
        mask = np.tril(np.ones((d, d), bool)) if uplo == "l" else np.triu(np.ones((d, d), bool))
        a = np.where(mask, vals, np.nan)  # the unreferenced triangle must never be read
        x, y = naive.fill(rng, d, tag), naive.fill(rng, d, tag)
        want, bound = cli.check_symv(uplo, herm, 0.75, a, x, 1.25, y, np.finfo(naive.DTYPES[tag]).eps, panel=512)
        ref = naive.naive_symv_hemv(0.75, np.where(mask, vals, 0), uplo, x, 1.25, y, hermitian=herm)
        assert np.all(np.isfinite(want))
        assert np.max(np.abs(want - ref)) <= bound

    def test_argument_errors(self):
        assert cli.main(["run", "--kernel", "hemv", "--prec", "d", "--n", "8"]) == 2
        assert cli.main(["run", "--kernel", "symv", "--n", "8", "--row-off", "1", "--col-off", "2"]) == 2
        assert cli.main(["run", "--kernel", "gemv", "--n", "0"]) == 2
        assert cli.main(["run", "--kernel", "gemv", "--n", "8", "--devices", "2", "--row-off", "1"]) == 2

    def test_copy_peak_env(self, monkeypatch):
        monkeypatch.setenv("KBLAS_COPY_PEAK_GBS", "1234.5")
        assert cli.copy_peak() == (1234.5, "env")


@pytest.mark.gpu
class TestRunGpu:
    @pytest.mark.parametrize("argv", [
        ["--kernel", "gemv", "--prec", "d", "--n", "700", "--m", "500"],
        ["--kernel", "gemv-t", "--prec", "s", "--n", "1000"],
        ["--kernel", "gemv-c", "--prec", "z", "--n", "300", "--row-off", "7", "--col-off", "3"],
        ["--kernel", "symv", "--prec", "d", "--n", "1100", "--uplo", "u"],
        ["--kernel", "hemv", "--prec", "c", "--n", "900", "--row-off", "13"],
        ["--kernel", "symv", "--prec", "d", "--n", "1000", "--devices", "3", "--nb", "64"],
        ["--kernel", "gemv", "--prec", "z", "--n", "600", "--devices", "2", "--beta", "0"],
    ])
    def test_run_verifies(self, tmp_path, argv):
        out = tmp_path / "run.csv"
        rc = cli.main(["run", *argv, "--reps", "3", "--warmup", "1", "--csv", str(out)])
        assert rc == 0
        rows = list(csv.DictReader(open(out)))
        merged = rows[0]
        assert merged["scope"] == "merged" and merged["verified"] == "pass"
        assert float(merged["achieved_gbs"]) > 0 and float(merged["measured_seconds"]) > 0
        devices = int(merged["devices"])
        assert len(rows) == 1 + (devices if devices > 1 else 0)


class TestRooflineTable:
    """`roofline` mirrors the reference's intensity table (test_cli.py:90-110):
    8 rows, intensity exact at the sample size, peak = intensity x the copy
    bandwidth."""

    def test_eight_rows(self, tmp_path, monkeypatch):
        monkeypatch.setenv("KBLAS_COPY_PEAK_GBS", "100")
        out = tmp_path / "roofline.csv"
        assert cli.main(["roofline", "--csv", str(out)]) == 0
        rows = list(csv.reader(open(out)))
        assert rows[0] == ["precision", "family", "n", "flops", "bytes", "intensity", "peak_gflops", "note"]
        assert len(rows) == 9
        s_gemv = next(r for r in rows[1:] if r[0] == "s" and r[1] == "gemv")
        assert float(s_gemv[5]) == pytest.approx(0.50, abs=5e-6)
        assert float(s_gemv[6]) == pytest.approx(50.0, abs=0.01)
        z_symv = next(r for r in rows[1:] if r[0] == "z" and r[1] == "symv")
        assert float(z_symv[5]) == pytest.approx(1.0, abs=1e-5)


class TestOffsetScanArgs:
    def test_errors(self):
        assert cli.main(["offset-scan", "--n", "0"]) == 2
        assert cli.main(["offset-scan", "--max-off", "-1"]) == 2


@pytest.mark.gpu
class TestOffsetScanGpu:
    @pytest.mark.parametrize("kernel", ["gemv", "gemv-t"])
    @pytest.mark.parametrize("tag", "dz")
    def test_scan(self, tmp_path, kernel, tag):
        out = tmp_path / "scan.csv"
        assert cli.main(["offset-scan", "--kernel", kernel, "--prec", tag, "--n", "1024", "--max-off", "33",
                         "--reps", "3", "--csv", str(out)]) == 0
        rows = list(csv.reader(open(out)))
        assert rows[0] == ["offset", "matrix_bytes", "measured_seconds", "achieved_gbs", "inflation"]
        assert [int(r[0]) for r in rows[1:]] == list(range(34))
        assert float(rows[1][4]) == 1.0
        assert all(float(r[3]) > 0 for r in rows[1:])
