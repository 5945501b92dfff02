"""Command-line front end (SPEC.md "cli" module, :689-745) and the CSEQ1 signal
file format, on this package's device path.

    python -m paper_2302_06646_b200.cli convolve --input u.cseq --kernel k.cseq \\
        --output y.cseq [--skip d.cseq] [--engine butterfly|three_pass|auto] \\
        [--mode causal|circular] [--lambda 0.003] [--p 1] [--seed 0] [--precision fp32|bf16|fp16]
    python -m paper_2302_06646_b200.cli kernel init --kind geometric --heads H --len N \\
        --seed 3 --output k.cseq [--skip-output d.cseq]
    python -m paper_2302_06646_b200.cli kernel regularize --input k.cseq --lambda 0.003 --p 1 \\
        --output kbar.cseq
    python -m paper_2302_06646_b200.cli bench --n 4096,65536 --r 16 \\
        --engines butterfly,three_pass --repetitions 5 --output rows.csv

CSEQ1: the 8-byte magic "CSEQ0001", then B, H, N as little-endian uint64,
then B*H*N little-endian float64 (row-major, N innermost).  The CSV
alternative (header ``b,h,n,value``) is accepted and written when the path
ends in ``.csv``.  A kernel bank is a CSEQ1 file with B = 1 (H kernels of
length N); skip gains D, when given, a CSEQ1 file with B = 1, N = 1.
Parse failures and dimension mismatches exit with status 2 and a message
(naming the byte offset for truncated files); outputs are written to a
temporary file and renamed, so no partial output is left behind.
"""
from __future__ import annotations

import argparse
import csv
import os
import struct
import sys
import tempfile

import numpy as np

MAGIC = b"CSEQ0001"


class FormatError(ValueError):
    pass


def read_signal(path: str) -> np.ndarray:
    """CSEQ1 (or CSV b,h,n,value) -> float64 array [B, H, N]."""
    if path.endswith(".csv"):
        with open(path, newline="") as f:
            rows = list(csv.reader(f))
        if not rows or [c.strip() for c in rows[0]] != ["b", "h", "n", "value"]:
            raise FormatError(f"{path}: CSV header must be b,h,n,value")
        try:
            recs = [(int(b), int(h), int(n), float(v)) for b, h, n, v in rows[1:]]
        except ValueError as e:
            raise FormatError(f"{path}: bad CSV row ({e})") from None
        if not recs:
            raise FormatError(f"{path}: no data rows")
        B, H, N = (max(r[i] for r in recs) + 1 for i in range(3))
        out = np.zeros((B, H, N))
        for b, h, n, v in recs:
            out[b, h, n] = v
        return out
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 32:
        raise FormatError(f"{path}: truncated header at byte offset {len(data)} (need 32)")
    if data[:8] != MAGIC:
        raise FormatError(f"{path}: bad magic at byte offset 0 (expected CSEQ0001)")
    B, H, N = struct.unpack_from("<QQQ", data, 8)
    need = 32 + 8 * B * H * N
    if len(data) < need:
        raise FormatError(f"{path}: truncated payload at byte offset {len(data)} (need {need})")
    if len(data) > need:
        raise FormatError(f"{path}: trailing bytes at byte offset {need}")
    return np.frombuffer(data, dtype="<f8", offset=32).reshape(B, H, N).astype(np.float64)


def write_signal(path: str, x: np.ndarray) -> None:
    """[B, H, N] -> CSEQ1 (or CSV by extension), atomically."""
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 3:
        raise FormatError("signals are [B, H, N]")
    d = os.path.dirname(os.path.abspath(path))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".cseq-")
    try:
        with os.fdopen(fd, "wb" if not path.endswith(".csv") else "w", **({} if not path.endswith(".csv")
                                                                         else {"newline": ""})) as f:
            if path.endswith(".csv"):
                w = csv.writer(f)
                w.writerow(["b", "h", "n", "value"])
                for (b, h, n), v in np.ndenumerate(x):
                    w.writerow([b, h, n, repr(float(v))])
            else:
                f.write(MAGIC + struct.pack("<QQQ", *x.shape) + x.astype("<f8").tobytes())
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _dtype(name):
    import torch

    return {"fp32": torch.float32, "bf16": torch.bfloat16, "fp16": torch.float16}[name]


def cmd_convolve(a) -> int:
    import torch

    from . import longconv as lc

    u = read_signal(a.input)
    k = read_signal(a.kernel)
    if k.shape[0] != 1 or k.shape[1:] != u.shape[1:]:
        raise FormatError(f"kernel bank {list(k.shape)} does not match the input's H, N {list(u.shape[1:])}")
    H, N = u.shape[1:]
    if a.skip:
        d = read_signal(a.skip)
        if d.shape != (1, H, 1):
            raise FormatError(f"skip gains must be [1, {H}, 1], got {list(d.shape)}")
        D = d[0, :, 0]
    else:
        D = np.zeros(H)
    dev = torch.device("cuda", a.device)
    dt = _dtype(a.precision)
    engine = {"butterfly": lc.Engine.BUTTERFLY, "three_pass": lc.Engine.THREE_PASS, "auto": lc.Engine.AUTO}[a.engine]
    mode = lc.ConvMode.CAUSAL if a.mode == "causal" else lc.ConvMode.CIRCULAR
    cfg = lc.RegularizationConfig(lambda_=a.lam, smooth_width=a.p, seed=a.seed)
    y = lc.regularized_long_conv(torch.tensor(u, dtype=dt, device=dev), torch.tensor(k[0], device=dev),
                                 torch.tensor(D, device=dev), cfg, engine, mode)
    write_signal(a.output, y.double().cpu().numpy())
    return 0


def cmd_kernel(a) -> int:
    import torch

    from . import longconv as lc

    dev = torch.device("cuda", a.device)
    if a.action == "init":
        kind = lc.InitKind.GEOMETRIC if a.kind == "geometric" else lc.InitKind.RANDOM
        K, D = lc.init_kernels(kind, a.heads, a.len, a.seed, dev, dtype=torch.float64)
        write_signal(a.output, K.cpu().numpy()[None])
        if a.skip_output:
            write_signal(a.skip_output, D.cpu().numpy()[None, :, None])
        return 0
    k = read_signal(a.input)
    if k.shape[0] != 1:
        raise FormatError("a kernel bank file has B = 1")
    H, N = k.shape[1:]
    plan = lc.LongConvPlan(N, H, lc.ConvMode.CAUSAL, torch.float32, lc.Engine.AUTO, dev)
    plan.prep(torch.tensor(k[0], device=dev), torch.zeros(H, device=dev),
              lc.RegularizationConfig(lambda_=a.lam, smooth_width=a.p, dropout_rate=a.dropout, seed=a.seed),
              training=a.dropout > 0)
    write_signal(a.output, plan.kbar().double().cpu().numpy()[None])
    return 0


def cmd_bench(a) -> int:
    """BenchRow CSV (SPEC.md cli): engine, n, l, m, r, repetitions, median wall
    time (ns, CUDA events around one layer forward at B = 1, H = 1 ... the
    --batch / --heads given), passes over the sequence (the engine's
    structure: 1 single-pass, 3 three-pass), and the flop model (40 sum(f) E)."""
    import torch

    from . import longconv as lc

    dev = torch.device("cuda", a.device)
    ns = [int(v) for v in a.n.split(",")]
    rs = [int(v) for v in a.r.split(",")]
    engines = a.engines.split(",")
    rows = []
    for eng in engines:
        e = {"butterfly": lc.Engine.BUTTERFLY, "three_pass": lc.Engine.THREE_PASS, "auto": lc.Engine.AUTO}[eng]
        for n in ns:
            N = n // 2
            for r in rs:
                try:
                    plan = lc.LongConvPlan(N, a.heads, lc.ConvMode.CAUSAL, _dtype(a.precision), e, dev)
                except Exception as ex:  # inadmissible (n, engine): a warning row
                    rows.append([eng, n, "", "", r, 0, "", "", "", f"skipped: {ex}"])
                    continue
                K = torch.randn(a.heads, N, device=dev) * 0.01
                plan.prep(K, torch.zeros(a.heads, device=dev), lc.RegularizationConfig())
                u = torch.randn(a.batch, a.heads, N, device=dev).to(_dtype(a.precision))
                for _ in range(2):
                    plan.forward(u)
                times = []
                for _ in range(max(3, a.repetitions)):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    plan.forward(u)
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e6)
                f, seg = [], n
                while seg > 1:  # build_plan(n, r) greedy chain (butterfly.cpp:83-100)
                    d = seg if seg <= r else next((d for d in range(min(seg, r), 1, -1) if seg % d == 0), 0)
                    if not d:
                        break
                    f.append(d)
                    seg //= d
                E = a.batch * a.heads * N
                rows.append([eng, n, plan.l, plan.m, r, len(times), int(np.median(times)),
                             3 if plan.m > 1 else 1, 40 * sum(f) * E, ""])
    hdr = ["engine", "n", "l", "m", "r", "repetitions", "median_wall_time_ns", "passes", "theoretical_flops",
           "note"]
    d = os.path.dirname(os.path.abspath(a.output))
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".bench-")
    with os.fdopen(fd, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(hdr)
        w.writerows(rows)
    os.replace(tmp, a.output)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2302_06646_b200.cli")
    ap.add_argument("--device", type=int, default=0)
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("convolve")
    c.add_argument("--input", required=True)
    c.add_argument("--kernel", required=True)
    c.add_argument("--output", required=True)
    c.add_argument("--skip")
    c.add_argument("--engine", default="butterfly", choices=["butterfly", "three_pass", "auto"])
    c.add_argument("--mode", default="causal", choices=["causal", "circular"])
    c.add_argument("--lambda", dest="lam", type=float, default=0.0)
    c.add_argument("--p", type=int, default=0)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--precision", default="fp32", choices=["fp32", "bf16", "fp16"])
    k = sub.add_parser("kernel")
    k.add_argument("action", choices=["init", "regularize"])
    k.add_argument("--kind", default="geometric", choices=["random", "geometric"])
    k.add_argument("--heads", type=int, default=1)
    k.add_argument("--len", type=int, default=1)
    k.add_argument("--seed", type=int, default=0)
    k.add_argument("--input")
    k.add_argument("--output", required=True)
    k.add_argument("--skip-output")
    k.add_argument("--lambda", dest="lam", type=float, default=0.0)
    k.add_argument("--p", type=int, default=0)
    k.add_argument("--dropout", type=float, default=0.0)
    b = sub.add_parser("bench")
    b.add_argument("--n", required=True, help="transform lengths n = 2N, comma separated")
    b.add_argument("--r", default="16")
    b.add_argument("--engines", default="butterfly")
    b.add_argument("--repetitions", type=int, default=5)
    b.add_argument("--batch", type=int, default=1)
    b.add_argument("--heads", type=int, default=1)
    b.add_argument("--precision", default="fp32", choices=["fp32", "bf16", "fp16"])
    b.add_argument("--output", required=True)
    a = ap.parse_args(argv)
    try:
        return {"convolve": cmd_convolve, "kernel": cmd_kernel, "bench": cmd_bench}[a.cmd](a)
    except FormatError as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
