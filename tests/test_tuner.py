"""The measured tuner and the library's tuning table (
reference tests/test_tuner.py:80-160 for the coarse/fine contract).

CPU: table set/get/replace/validation through the C ABI (host-only calls),
candidate enumeration, range construction, save/load and
$KBLAS_TUNING_FILE.  GPU: a tuned entry changes the kernel that runs (the
plan) and not the result; coarse/fine on small sizes."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1410_1726_b200 import _lib, tuner
from paper_1410_1726_b200.core import precision

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture
def clean_table():
    saved = tuner.table()
    tuner.clear()
    yield
    tuner.restore(saved)


class TestTable:
    def test_set_get_replace(self, clean_table):
        tuner.set_entry(tuner.TableEntry("d", "n", 100, 200, 3, 1, 2))
        tuner.set_entry(tuner.TableEntry("z", "l", 1000, 2000, 105))
        assert tuner.table() == [tuner.TableEntry("d", "n", 100, 200, 3, 1, 2),
                                 tuner.TableEntry("z", "l", 1000, 2000, 105, -1, 0)]
        tuner.set_entry(tuner.TableEntry("d", "n", 100, 200, 4, 0, 0))  # same range: replaced
        assert tuner.table()[0] == tuner.TableEntry("d", "n", 100, 200, 4, 0, 0)
        assert len(tuner.table()) == 2
        tuner.clear()
        assert tuner.table() == []

    def test_case_insensitive(self, clean_table):
        assert _lib.load().kblas_tune_set(b"D", b"T", 1, 2, 5, 1, 0) == 0
        assert tuner.table() == [tuner.TableEntry("d", "t", 1, 2, 5, 1, 0)]

    @pytest.mark.parametrize("args,k", [
        ((b"x", b"n", 1, 2, 0, -1, 0), 1),
        ((b"d", b"q", 1, 2, 0, -1, 0), 2),
        ((b"d", b"n", -1, 2, 0, -1, 0), 3),
        ((b"d", b"n", 5, 2, 0, -1, 0), 4),
        ((b"d", b"n", 1, 2, 7, -1, 0), 5),      # not a GEMV shape
        ((b"d", b"n", 1, 2, 5, 3, 0), 5),       # row-owning needs a configuration shape 10..17
        ((b"d", b"n", 1, 2, 18, 3, 0), 5),
        ((b"d", b"t", 1, 2, 12, 1, 0), 5),
        ((b"d", b"l", 1, 2, 3, -1, 0), 5),      # a GEMV shape for SYMV
        ((b"d", b"n", 1, 2, 0, 4, 0), 6),       # GEMV-N forms are -1..3
        ((b"d", b"t", 1, 2, 0, 2, 0), 6),       # GEMV-T forms are -1..1
        ((b"d", b"l", 1, 2, 100, 0, 0), 6),     # SYMV has no form
        ((b"d", b"t", 1, 2, 0, -1, 2), 7),      # waves only for GEMV-N
        ((b"d", b"n", 1, 2, 0, -1, 65), 7),
    ])
    def test_invalid_arguments(self, clean_table, args, k):
        assert _lib.load().kblas_tune_set(*args) == -k
        assert tuner.table() == []
        with pytest.raises(ValueError, match=f"invalid argument {k}"):
            tuner.set_entry(tuner.TableEntry(args[0].decode(), args[1].decode(), *args[2:]))

    def test_get_out_of_range(self):
        assert _lib.load().kblas_tune_get(10 ** 6, None, None, None, None, None, None, None) == -1


class TestEnumerate:
    def test_builtin_first(self):
        for k in tuner.KERNELS:
            for stage in ("coarse", "fine"):
                c = tuner.enumerate_configs(k, stage)
                assert c[0].is_auto and len(set(c)) == len(c)

    def test_shapes_and_forms(self):
        assert [c.shape for c in tuner.enumerate_configs("gemv")[1:]] == list(tuner.GEMV_SHAPES)
        assert {c.form for c in tuner.enumerate_configs("gemv-t")[1:]} == {0}
        fine = tuner.enumerate_configs("gemv", "fine", 3)
        assert {(c.form, c.waves) for c in fine[1:] if c.shape == 3} == {(0, 0), (1, 0), (2, 0), (1, 2), (-1, 0)}
        assert {(c.form, c.waves) for c in fine[1:] if c.shape == 0} == {(0, 0), (1, 0), (2, 0), (1, 2)}
        assert {c.shape for c in fine if c.form == 3} == set(range(10, 18))
        assert {c.shape for c in fine} == {0, 3} | set(range(10, 18))
        assert {(c.shape, c.form) for c in tuner.enumerate_configs("gemv-c", "fine", 5)[1:]} == {
            (5, 0), (5, 1), (5, -1), (0, 0), (0, 1)}
        assert {c.shape for c in tuner.enumerate_configs("gemv-t", "fine")} == {0}
        assert [c.shape for c in tuner.enumerate_configs("hemv", "fine")[1:]] == list(tuner.SYMV_SHAPES)

    def test_errors(self):
        with pytest.raises(ValueError):
            tuner.enumerate_configs("gemm")
        with pytest.raises(ValueError):
            tuner.enumerate_configs("gemv", "medium")
        with pytest.raises(ValueError):
            tuner.op_of("symv", "x")
        with pytest.raises(ValueError):
            tuner._check_kernel("hemv", precision("d"))
        with pytest.raises(ValueError):
            tuner.coarse_tune("gemv", precision("d"), [])
        with pytest.raises(ValueError):
            tuner.fine_tune("gemv", precision("d"), [])


class TestRanges:
    def _fine(self, kernel, per_size, uplo="l", tag="d"):
        return tuner.FineResult(kernel, precision(tag), uplo, per_size, per_size[max(per_size)])

    def test_nearest_size_cover(self):
        A = tuner.TuneConfig(5, 1)
        B = tuner.TuneConfig(3, 0)
        rows = tuner.entries_for(self._fine("gemv", {1024: A, 4096: B, 16384: A}))
        assert [(r.n_lo, r.n_hi, r.shape, r.form) for r in rows] == [
            (725, 2048, 5, 1), (2049, 8192, 3, 0), (8193, 23170, 5, 1)]
        assert all(r.op == "n" and r.prec == "d" for r in rows)

    def test_builtin_winner_adds_nothing(self):
        auto = tuner.auto_config("symv")
        rows = tuner.entries_for(self._fine("hemv", {2048: auto, 8192: tuner.TuneConfig(105)}, "u", "z"))
        assert [(r.op, r.n_lo, r.n_hi, r.shape) for r in rows] == [("u", 4097, 11585, 105)]

    def test_single_size(self):
        rows = tuner.entries_for(self._fine("gemv-c", {4096: tuner.TuneConfig(0, 1)}, tag="z"))
        assert [(r.op, r.n_lo, r.n_hi) for r in rows] == [("c", 2897, 5792)]


class TestSaveLoad:
    def test_round_trip(self, clean_table, tmp_path):
        rows = [tuner.TableEntry("s", "n", 10, 20, 4, 2, 0), tuner.TableEntry("c", "u", 1, 5, 103)]
        for r in rows:
            tuner.set_entry(r)
        path = str(tmp_path / "t.json")
        tuner.save(path, device="test")
        tuner.clear()
        assert tuner.load(path) == 2
        assert tuner.table() == rows
        assert tuner.load(path, replace=True) == 2
        assert tuner.table() == rows
        doc = json.load(open(path))
        assert doc["device"] == "test" and doc["format"] == "kblas-b200-tuning/1"

    def test_merge_replaces_only_the_retuned_kernel(self):
        old = [tuner.TableEntry("d", "n", 1, 10, 3, 0), tuner.TableEntry("z", "l", 1, 10, 105),
               tuner.TableEntry("d", "t", 1, 10, 0, 1)]
        fine = tuner.FineResult("gemv", precision("d"), "l", {2048: tuner.TuneConfig(11, 3)},
                                tuner.TuneConfig(11, 3))
        merged = tuner.merge_entries(old, fine)
        assert merged[:2] == [old[1], old[2]]
        assert [(e.prec, e.op, e.shape, e.form) for e in merged[2:]] == [("d", "n", 11, 3)]

    def test_read_does_not_install(self, clean_table, tmp_path):
        path = str(tmp_path / "t.json")
        tuner.save(path, [tuner.TableEntry("s", "n", 10, 20, 4, 2, 0)])
        assert tuner.read(path) == [tuner.TableEntry("s", "n", 10, 20, 4, 2, 0)]
        assert tuner.table() == []

    def test_bad_file(self, clean_table, tmp_path):
        p = tmp_path / "bad.json"
        p.write_text(json.dumps({"format": "other", "entries": []}))
        with pytest.raises(ValueError, match="not a kblas-b200 tuning table"):
            tuner.load(str(p))

    def test_env_file_loaded_at_library_load(self, tmp_path):
        path = tmp_path / "t.json"
        path.write_text(json.dumps({"format": "kblas-b200-tuning/1", "device": None, "entries": [
            {"prec": "z", "op": "n", "n_lo": 3000, "n_hi": 5000, "shape": 3, "form": 2, "waves": 0}]}))
        code = ("from paper_1410_1726_b200 import tuner; "
                "print([tuple(e.__dict__.values()) for e in tuner.table()])")
        env = dict(os.environ, KBLAS_TUNING_FILE=str(path), PYTHONPATH=ROOT)
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
        assert out.returncode == 0, out.stderr
        assert "('z', 'n', 3000, 5000, 3, 2, 0)" in out.stdout

    def test_env_file_invalid_entry_fails_loudly(self, tmp_path):
        path = tmp_path / "t.json"
        path.write_text(json.dumps({"format": "kblas-b200-tuning/1", "entries": [
            {"prec": "d", "op": "l", "n_lo": 1, "n_hi": 2, "shape": 3}]}))
        env = dict(os.environ, KBLAS_TUNING_FILE=str(path), PYTHONPATH=ROOT)
        out = subprocess.run([sys.executable, "-c", "from paper_1410_1726_b200 import _lib; _lib.load()"],
                             env=env, capture_output=True, text=True, cwd=ROOT)
        assert out.returncode != 0 and "invalid argument 5" in out.stderr


# ----------------------------------------------------------------------- GPU
def _gemv_call(tag, trans, n, seed=0):
    import torch

    import paper_1410_1726_b200 as kb

    p = precision(tag)
    g = torch.Generator(device="cuda").manual_seed(seed)

    def rnd(*shape):
        t = torch.empty(*shape, dtype=p.torch_dtype, device="cuda")
        (torch.view_as_real(t) if p.is_complex else t).uniform_(-1, 1, generator=g)
        return t

    A, x, y = rnd(n, n), rnd(n), rnd(n)
    view = kb.view_of(A.T)  # column-major n x n
    return lambda: (kb.gemv(trans, 1.0, view, x, 0.5, y).y_out.cpu().numpy(), _lib.last_plan())


def _symv_call(tag, uplo, n, herm, seed=0):
    import torch

    import paper_1410_1726_b200 as kb

    p = precision(tag)
    g = torch.Generator(device="cuda").manual_seed(seed)

    def rnd(*shape):
        t = torch.empty(*shape, dtype=p.torch_dtype, device="cuda")
        (torch.view_as_real(t) if p.is_complex else t).uniform_(-1, 1, generator=g)
        return t

    A, x, y = rnd(n, n), rnd(n), rnd(n)
    hv = kb.HermitianView(kb.view_of(A.T), uplo)
    return lambda: (kb.symv_hemv(uplo, 1.0, hv, x, 0.5, y, hermitian=herm).y_out.cpu().numpy(), _lib.last_plan())


def _close(a, b, tag, n):
    scale = max(1.0, float(np.abs(b).max()))
    assert float(np.abs(a - b).max()) <= 64 * precision(tag).eps * np.sqrt(n) * scale


@pytest.mark.gpu
class TestTableDrivesDispatch:
    @pytest.mark.parametrize("tag", "dz")
    def test_gemv_n_forms(self, clean_table, tag):
        n = 3000
        run = _gemv_call(tag, "n", n)
        y0, plan0 = run()
        seen = {}
        for form, prefix in ((0, "gemv_n "), (1, "gemv_ns "), (2, "gemv_nc "), (3, "gemv_ro ")):
            tuner.clear()
            # row-owning config 7 (16 / 32 rows per CTA): one wave at n = 3000,
            # so the form's wave guard accepts it (config 1 takes 1.3 waves for z)
            tuner.set_entry(tuner.TableEntry(tag, "n", n - 10, n + 10, 17 if form == 3 else 5, form, 0))
            y, plan = run()
            assert plan.startswith(prefix), (form, plan)
            _close(y, y0, tag, n)
            seen[form] = plan
        # outside the entry's range the built-in rule runs again
        tuner.clear()
        tuner.set_entry(tuner.TableEntry(tag, "n", n + 1, n + 10, 5, 0, 0))
        _, plan = run()
        assert plan == plan0

    @pytest.mark.parametrize("tag,trans", [("d", "t"), ("c", "c"), ("s", "c")])
    def test_gemv_t_forms(self, clean_table, tag, trans):
        n = 2500
        run = _gemv_call(tag, trans, n)
        y0, _ = run()
        for form, prefix in ((0, "gemv_t "), (1, "gemv_tc ")):
            tuner.clear()
            # the table key of 'c' on a real precision is 't'
            op = "t" if (trans == "c" and tag in "sd") else trans
            tuner.set_entry(tuner.TableEntry(tag, op, 0, 10 ** 6, 4, form, 0))
            y, plan = run()
            assert plan.startswith(prefix), (form, plan)
            _close(y, y0, tag, n)

    def test_rowown_declined_falls_back_to_rules(self, clean_table):
        """A short, wide matrix keyed into a row-owning range has too few
        row blocks for it: the call runs what the built-in rules pick."""
        import torch

        import paper_1410_1726_b200 as kb

        m, n = 64, 65536
        A = torch.empty(n, m, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        v = kb.view_of(A.T)
        x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
        y = torch.zeros(m, dtype=torch.float64, device="cuda")
        r0 = kb.gemv("n", 1.0, v, x, 0.0, y)
        tuner.set_entry(tuner.TableEntry("d", "n", 1000, 5000, 11, 3, 0))  # key sqrt(64*65536) = 2048
        r1 = kb.gemv("n", 1.0, v, x, 0.0, y)
        assert r1.plan == r0.plan and not r1.plan.startswith("gemv_ro")
        assert torch.equal(r0.y_out, r1.y_out)

    def test_setter_wins_over_table(self, clean_table):
        n = 3000
        run = _gemv_call("d", "n", n)
        tuner.set_entry(tuner.TableEntry("d", "n", 0, 10 ** 6, 5, 0, 0))
        prev = _lib.set_gemv_split(1)
        try:
            _, plan = run()
            assert plan.startswith(("gemv_ns ", "gemv_nc ")), plan
        finally:
            _lib.set_gemv_split(prev)

    @pytest.mark.parametrize("tag,herm", [("d", False), ("z", True), ("c", False)])
    @pytest.mark.parametrize("uplo", "lu")
    def test_symv_shapes(self, clean_table, tag, herm, uplo):
        n = 2600
        run = _symv_call(tag, uplo, n, herm)
        prev = _lib.set_tma(0)
        try:
            y0, _ = run()
            widths = {}
            for shape in tuner.SYMV_SHAPES:
                tuner.clear()
                tuner.set_entry(tuner.TableEntry(tag, uplo, n, n, shape))
                y, plan = run()
                _close(y, y0, tag, n)
                widths[shape] = [w for w in plan.split() if w.startswith("W=")][0]
            assert widths[103] != widths[100]
        finally:
            _lib.set_tma(prev)


@pytest.mark.gpu
class TestTuner:
    def test_coarse_fine_gemv(self, clean_table):
        coarse, fine = tuner.tune("gemv", "d", [1024, 3000], reps=3, warmup=1)
        assert coarse.winner in tuner.enumerate_configs("gemv", "coarse")
        assert set(fine.per_size) == {1024, 3000}
        assert fine.recommended == fine.per_size[3000]
        assert all(p.measured_gbs > 0 and p.rel_diff <= 64 * 2.3e-16 * np.sqrt(p.size) for p in fine.points)
        assert tuner.table() == []  # measuring leaves the table as it was
        rows = tuner.apply(fine)
        assert tuner.table() == rows

    def test_symv_sweep_and_csv(self, clean_table, tmp_path):
        tuner.set_entry(tuner.TableEntry("z", "l", 5, 6, 105))
        coarse, fine = tuner.tune("hemv", "z", [1500], reps=3, warmup=1)
        assert tuner.table() == [tuner.TableEntry("z", "l", 5, 6, 105)]
        path = tmp_path / "s.csv"
        with open(path, "w") as fh:
            tuner.write_sweep_csv(coarse.points + fine.points, fh)
        lines = path.read_text().splitlines()
        assert lines[0].split(",") == tuner.SWEEP_CSV_HEADER
        assert len(lines) == 1 + len(coarse.points) + len(fine.points)

    def test_cli_tune_save(self, clean_table, tmp_path):
        from paper_1410_1726_b200 import cli

        out = tmp_path / "table.json"
        assert cli.main(["tune", "--kernel", "gemv-t", "--prec", "z", "--sizes", "1024,2048", "--reps", "3",
                         "--csv", str(tmp_path / "t.csv"), "--save", str(out)]) == 0
        doc = json.loads(out.read_text())
        assert doc["format"] == "kblas-b200-tuning/1"
        assert all(e["prec"] == "z" and e["op"] == "t" for e in doc["entries"])  # no built-in rows
        # --merge keeps the file's other kernels
        assert cli.main(["tune", "--kernel", "hemv", "--prec", "z", "--sizes", "1024", "--reps", "3",
                         "--csv", str(tmp_path / "h.csv"), "--save", str(out), "--merge"]) == 0
        doc2 = json.loads(out.read_text())
        assert {(e["prec"], e["op"]) for e in doc2["entries"]} <= {("z", "t"), ("z", "l")}
        assert [e for e in doc2["entries"] if e["op"] == "t"] == doc["entries"]


class TestBuiltinTable:
    def test_matches_shipped_json(self, clean_table):
        assert tuner.defaults() == len(tuner.table())
        doc = json.load(open(tuner.BUILTIN_TABLE))
        assert doc["format"] == "kblas-b200-tuning/1"
        assert tuner.table() == [tuner.TableEntry(**e) for e in doc["entries"]]

    def test_ranges_disjoint_per_op(self):
        doc = json.load(open(tuner.BUILTIN_TABLE))
        by = {}
        for e in doc["entries"]:
            by.setdefault((e["prec"], e["op"]), []).append((e["n_lo"], e["n_hi"]))
        for rs in by.values():
            rs.sort()
            assert all(a[1] < b[0] for a, b in zip(rs, rs[1:]))


@pytest.mark.gpu
class TestShippedTableGuards:
    """The shipped table together with the dispatch guards."""

    def test_rowown_wave_guard(self):
        # D GEMV-N 3548..5016 is a row-owning row (config 1: 16 rows per CTA
        # of 8 warps).  At P = 290 CTAs the grid is one wave on a B200 and
        # the form runs; at P = 302 the last wave would hold 6 CTAs and the
        # guard hands the call to the built-in rule.
        _, plan_in = _gemv_call("d", "n", 290 * 16)()
        _, plan_out = _gemv_call("d", "n", 302 * 16)()
        assert plan_in.startswith("gemv_ro "), plan_in
        assert not plan_out.startswith("gemv_ro "), plan_out

    @pytest.mark.parametrize("trans", ["t", "c"])
    def test_c_column_owning_rows(self, trans):
        _, plan = _gemv_call("c", trans, 24576)()
        assert plan.startswith("gemv_tc "), plan

    def test_z_cluster_rows_stop_at_the_cliff(self):
        _, below = _gemv_call("z", "n", 4224)()
        _, above = _gemv_call("z", "n", 4288)()
        assert below.startswith("gemv_nc "), below
        assert not above.startswith("gemv_nc "), above
