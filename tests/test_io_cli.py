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
