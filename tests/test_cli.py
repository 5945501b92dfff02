"""The CSEQ1 file format and the command-line front end
(SPEC.md cli module): parsing / atomic writes on CPU, the device commands on
the B200 against the fp64 oracle."""
import os
import struct

import numpy as np
import pytest

from paper_2302_06646_b200 import cli
from oracle.oracle import rel_l2


def test_cseq1_round_trip(tmp_path):
    x = np.random.default_rng(0).standard_normal((2, 3, 5))
    p = str(tmp_path / "x.cseq")
    cli.write_signal(p, x)
    raw = open(p, "rb").read()
    assert raw[:8] == b"CSEQ0001" and struct.unpack_from("<QQQ", raw, 8) == (2, 3, 5)
    assert len(raw) == 32 + 8 * 30
    assert np.array_equal(cli.read_signal(p), x)
    c = str(tmp_path / "x.csv")
    cli.write_signal(c, x)
    assert open(c).readline().strip() == "b,h,n,value"
    assert np.array_equal(cli.read_signal(c), x)


def test_cseq1_errors(tmp_path):
    p = str(tmp_path / "t.cseq")
    cli.write_signal(p, np.ones((1, 2, 4)))
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-5])
    with pytest.raises(cli.FormatError, match="byte offset"):
        cli.read_signal(p)
    open(p, "wb").write(b"XSEQ0001" + raw[8:])
    with pytest.raises(cli.FormatError, match="magic"):
        cli.read_signal(p)


def test_convolve_parse_failure_leaves_no_output(tmp_path):
    u = str(tmp_path / "u.cseq")
    k = str(tmp_path / "k.cseq")
    y = str(tmp_path / "y.cseq")
    cli.write_signal(u, np.ones((1, 1, 8)))
    open(k, "wb").write(b"CSEQ0001" + struct.pack("<QQQ", 1, 1, 8) + b"\0" * 16)  # truncated
    assert cli.main(["convolve", "--input", u, "--kernel", k, "--output", y]) == 2
    assert not os.path.exists(y)


@pytest.mark.gpu
def test_convolve_delta_identity_and_oracle(tmp_path, lc):
    B, H, N = 2, 3, 1024
    u = lc.signal_batch(1, B, H, N).astype(np.float32).astype(np.float64)
    delta = np.zeros((1, H, N))
    delta[:, :, 0] = 1.0
    pu, pk, py = (str(tmp_path / f) for f in ("u.cseq", "k.cseq", "y.cseq"))
    cli.write_signal(pu, u)
    cli.write_signal(pk, delta)
    assert cli.main(["convolve", "--input", pu, "--kernel", pk, "--output", py]) == 0
    # identity layer (lambda = 0, p = 0); fp32 transforms, so 1e-5 rather than fp64's 1e-12
    assert rel_l2(cli.read_signal(py), u) < 1e-6 and np.abs(cli.read_signal(py) - u).max() < 1e-5
    K, D = lc.init_kernels(1, H, N, 3)
    K = K.astype(np.float32).astype(np.float64)
    D = D.astype(np.float32).astype(np.float64)
    pd = str(tmp_path / "d.cseq")
    cli.write_signal(pk, K[None])
    cli.write_signal(pd, D[None, :, None])
    assert cli.main(["convolve", "--input", pu, "--kernel", pk, "--skip", pd, "--output", py,
                     "--lambda", "0.003", "--p", "1"]) == 0
    want = lc.regularized_long_conv(u, K, D, 0.003, 1)
    assert rel_l2(cli.read_signal(py), want) < 1e-5


@pytest.mark.gpu
def test_kernel_init_and_bench(tmp_path, lc):
    pk, pd, pr = (str(tmp_path / f) for f in ("k.cseq", "d.cseq", "rows.csv"))
    assert cli.main(["kernel", "init", "--kind", "geometric", "--heads", "4", "--len", "300", "--seed", "3",
                     "--output", pk, "--skip-output", pd]) == 0
    K, D = lc.init_kernels(1, 4, 300, 3)
    assert rel_l2(cli.read_signal(pk)[0], K) < 1e-13
    assert rel_l2(cli.read_signal(pd)[0, :, 0], D) < 1e-13
    assert cli.main(["bench", "--n", "4096,32768", "--r", "16", "--engines", "butterfly,three_pass",
                     "--repetitions", "3", "--output", pr]) == 0
    rows = open(pr).read().strip().splitlines()
    assert rows[0].startswith("engine,n,l,m,r") and len(rows) == 5
