"""SFDT file ingest and the CLI: format validation on
the CPU; the GPU-backed CLI against the oracle."""

import json
import math

import numpy as np
import pytest

from paper_1407_8315_b200 import io as sio
from paper_1407_8315_b200.spectral import SparseSpectrum


def test_signal_round_trip_and_errors(tmp_path):
    x = np.arange(8) + 1j * np.arange(8)[::-1]
    p = tmp_path / "s.sfdt"
    sio.write_signal(p, x)
    assert np.array_equal(sio.read_signal(p), x)
    raw = p.read_bytes()
    cases = {
        "bad magic": b"XXXX" + raw[4:],
        "unsupported version": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "expected": raw[:-1],
        "truncated header": raw[:10],
    }
    for msg, data in cases.items():
        q = tmp_path / "bad.sfdt"
        q.write_bytes(data)
        with pytest.raises(sio.FormatError, match=msg):
            sio.read_signal(q)
    q = tmp_path / "len.sfdt"
    sio.write_signal(q, np.zeros(6))
    with pytest.raises(sio.FormatError, match="power of two"):
        sio.read_signal(q)


def test_spectrum_json_round_trip(tmp_path):
    spec = SparseSpectrum(16, {3: 1 + 2j, 0: -0.5j})
    p = tmp_path / "spec.json"
    sio.write_spectrum(p, spec)
    rows = json.loads(p.read_text())
    assert [r["index"] for r in rows] == [0, 3]
    assert sio.read_spectrum(p, 16).entries == spec.entries
    p.write_text("{not json")
    with pytest.raises(sio.FormatError):
        sio.read_spectrum(p, 16)


@pytest.mark.gpu
def test_cli_against_oracle(tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import kernels as OK
    from oracle import solvers as OS
    from paper_1407_8315_b200 import cli
    from tests.synth import exact_signal, general_signal

    n, k = 1 << 16, 64
    x, _ = exact_signal(n, k, 0, "unit", synth="radix2")
    sig = tmp_path / "cfg1.sfdt"
    sio.write_signal(sig, x)
    out = tmp_path / "spec.json"
    tr = tmp_path / "trace.json"
    rc = cli.main(["transform-exact", str(sig), "--k", str(k), "--out", str(out),
                   "--trace-out", str(tr)])
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    want, wtr = OS.exact_iterative(x, k)
    assert rc == 0 and summary["recovered"] == len(want) and summary["full_success"]
    got = sio.read_spectrum(out, n).entries
    assert set(got) == set(want)
    assert all(abs(got[s] - v) <= 1e-9 * abs(v) for s, v in want.items())
    assert json.loads(tr.read_text())["iterations"] == wtr["iterations"]

    rc = cli.main(["transform-exact", str(sig), "--k", str(k), "--solver", "non-iterative",
                   "--n", str(n)])
    assert rc == 0
    assert cli.main(["transform-exact", str(sig), "--k", str(k), "--n", "1024"]) == 1

    rc = cli.main(["estimate-k", str(sig)])
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    est = OS.exact_estimate(x)
    assert rc == 0 and summary["k_hat"] == est["k_hat"] and summary["final_d"] == est["final_d"]

    ng, kg = 1 << 14, 16
    xg, _ = general_signal(ng, kg, 20.0, 5)
    sg = tmp_path / "g.sfdt"
    sio.write_signal(sg, xg)
    rc = cli.main(["transform-general", str(sg), "--k", str(kg), "--seed", "5"])
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    want, _ = OS.general(xg, kg, rng_seed=5)
    ref = OK.fft_radix2(xg) / ng
    est_dense = np.zeros(ng, complex)
    for s, v in want.items():
        est_dense[s] = v
    snr = 10 * math.log10(np.mean(np.abs(est_dense) ** 2) / np.mean(np.abs(ref - est_dense) ** 2))
    assert rc == 0 and summary["entries"] == len(want)
    assert abs(summary["snr_db"] - round(snr, 3)) <= 1e-3


@pytest.mark.gpu
def test_read_signals_device_batch(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    rng = np.random.default_rng(1)
    xs = [rng.standard_normal(256) + 1j * rng.standard_normal(256) for _ in range(3)]
    paths = []
    for i, x in enumerate(xs):
        p = tmp_path / f"{i}.sfdt"
        sio.write_signal(p, x)
        paths.append(p)
    X = sio.read_signals_device(paths)
    assert X.shape == (3, 256) and X.is_cuda
    assert np.array_equal(X.cpu().numpy(), np.stack(xs))


@pytest.mark.gpu
@pytest.mark.gpu
def test_device_fft_bitexact_long():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import kernels as OK
    from paper_1407_8315_b200.spectral import fft
    rng = np.random.default_rng(2)
    # smem-only, 1 register pass, the shared-memory pass B (2^17 .. 2^19), 3 register passes
    for n in (8, 4096, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 21):
        x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        got = fft(x)
        assert np.array_equal(got.view(np.uint64), OK.fft_radix2(x).view(np.uint64)), n
        got = fft(x, inverse=True)
        assert np.array_equal(got.view(np.uint64), OK.fft_radix2(x, True).view(np.uint64)), n


def test_cli_census_subcommand(tmp_path, capsys):
    """`census` (reference cli.py:184-208): host integer counting, the
    reference's summary keys and CSV / JSON row layout."""
    import csv

    from paper_1407_8315_b200 import cli
    from paper_1407_8315_b200.experiments import run_collision_census
    out = tmp_path / "census.csv"
    rc = cli.main(["census", "--n", "4096", "--k", "16", "--n-plus", "4", "8", "--trials", "50",
                   "--seed", "3", "--out", str(out), "--threads", "2"])
    summary = json.loads(capsys.readouterr().out)
    want = run_collision_census(4096, 16, [4, 8], trials=50, seed=3)
    assert rc == 0 and sorted(summary) == ["4", "8"]
    for key, res in want.items():
        got = summary[str(key)]
        assert got == {"p_signal_over": res["p_signal_over"], "bound_signal_over": res["bound_signal_over"],
                       "p_bin_over": res["p_bin_over"]}
    rows = list(csv.DictReader(open(out)))
    assert list(rows[0]) == ["n_plus", "d", "a", "probability"]
    assert len(rows) == sum(len(r["per_bin_probability"]) for r in want.values())
    assert float(rows[1]["probability"]) == float(want[4]["per_bin_probability"][1])
    outj = tmp_path / "census.json"
    assert cli.main(["census", "--n", "4096", "--k", "16", "--trials", "10", "--format", "json",
                     "--out", str(outj)]) == 0
    capsys.readouterr()
    assert json.loads(outj.read_text())[0].keys() == {"n_plus", "d", "a", "probability"}
    # incompatible oversampling ratio: the reference's ValueError -> exit code 1
    assert cli.main(["census", "--n", "4096", "--k", "16", "--n-plus", "3"]) == 1


@pytest.mark.gpu
def test_cli_bench_subcommand(tmp_path, capsys):
    """`bench` (reference cli.py:161-181): the named grids, each cell one GPU
    batch; report columns as the reference writes them."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1407_8315_b200 import cli
    out = tmp_path / "grid.json"
    assert cli.main(["bench", "--grid", "exact-small", "--trials", "3", "--format", "json", "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["name"] == "exact_grid" and rep["meta"]["k_values"] == [16, 32, 64]
    assert len(rep["rows"]) == 9 and all(r["perfect"] == 1 for r in rep["rows"])
    assert list(rep["rows"][0]) == ["n", "k", "mu", "a_max", "solver", "seed", "perfect", "recovered_fraction",
                                    "full_success", "fft_samples", "elapsed_s"]
    outc = tmp_path / "grid.csv"
    assert cli.main(["bench", "--grid", "general-desk", "--trials", "2", "--out", str(outc)]) == 0
    cells = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert len(cells) == 6 and cells[0]["trials"] == 2 and "mean_snr_out_db_prune" in cells[0]
    assert outc.read_text().startswith("n,n_over_k,k,snr_target_db")
