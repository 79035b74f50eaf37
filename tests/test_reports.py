"""the device memory reports keep the reference's CSV schemas.
tests/golden/reports.json holds the reference's own `rtpsim memtable / ledger /
sweep` output (commands.cpp:87-181, run through oracle/_ref); the formatters in
paper_2311_01635_b200/reports.py must reproduce it byte for byte when fed the
reference's numbers, and the device run (GPU test) must emit the same keys."""
import json
import os

import numpy as np
import pytest

from paper_2311_01635_b200 import reports

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ref():
    with open(os.path.join(HERE, "golden", "reports.json")) as fh:
        return json.load(fh)


def _rows(text):
    lines = text.strip().split("\n")
    return lines[0], [ln.split(",") for ln in lines[1:]]


@pytest.mark.parametrize("n", [2, 4])
def test_memtable_reproduces_the_reference(ref, n):
    text = ref[f"memtable_n{n}_rtp-inplace"]
    hdr, rows = _rows(text)
    assert hdr == reports.MEMTABLE_HEADER
    assert [r[0] for r in rows] == list(reports.STRATEGIES)
    by = {r[0]: [int(v) for v in r[2:]] for r in rows}
    A, WG = by["no-parallelism"][0], by["no-parallelism"][1]
    Ap = (by["pipeline-parallel"][0] - A) // n
    W = G = WG // 2  # memtable without literals: G = W = params x 8 (commands.cpp:96-99)
    assert reports.memtable_csv(n, W, G, A, Ap) == text


def test_table1_rtp_rows_match_reference_goldens(golden):
    led = golden("ledger")
    for st, name in ((5, "rtp"), (6, "rtp-inplace")):
        for N in (1, 2, 4, 8):
            assert list(reports.table1_memory(name, 1000, 2000, 300, 40, N)) == list(led[f"table1_s{st}_N{N}"])


@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("strategy", ["rtp-inplace", "rtp-outofplace"])
def test_ledger_and_sweep_formatters_reproduce_the_reference(ref, n, strategy):
    text = ref[f"ledger_n{n}_{strategy}"]
    hdr, rows = _rows(text)
    assert hdr == reports.LEDGER_HEADER
    pk = {}
    for r in rows:
        pk.setdefault((r[0], int(r[1])), {})[r[2]] = int(r[3])
    serial = pk[("serial", 1)]
    assert reports.ledger_csv(serial, [(strategy, n, pk[(strategy, n)])]) == text
    text = ref[f"sweep_n{n}_{strategy}"]
    hdr, rows = _rows(text)
    assert hdr == reports.SWEEP_HEADER
    pts = [(int(r[2]), dict(zip(reports.CATEGORIES, (int(v) for v in r[4:9]))), int(r[9])) for r in rows]
    assert reports.sweep_csv(strategy, n, pts) == text


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["rtp-inplace", "rtp-outofplace"])
def test_device_ledger_report_has_the_reference_keys(ref, strategy):
    """A device MLP run's ledger report: same header and (strategy, n,
    category) rows as the reference's; RTP duplicates no parameter or
    gradient bytes (analysis_test.cpp:162-164)."""
    import torch
    from paper_2311_01635_b200 import rtp
    n, h, f, rows = 2, 64, 256, 64

    def run(nw, mode):
        g = rtp.WorkerGroup(nw)
        m = rtp.RtpMlp(g, "mlp", h, f, "bf16", seed=42)
        m.set_rotation_mode(mode)
        m.begin_step()
        m.zero_grads()
        gen = torch.Generator(device="cuda").manual_seed(0)
        xs = [(torch.rand(rows // nw, h, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16) for _ in range(nw)]
        m.forward(xs)
        m.backward(xs)
        g.synchronize()
        led = [g.ledger(r) for r in range(nw)]
        m.close()
        g.close()
        return led
    serial = reports.peaks_by_category(run(1, "inplace")[0])
    mode = "inplace" if strategy == "rtp-inplace" else "outofplace"
    worst = max(run(n, mode), key=lambda d: d["peak_total"])
    text = reports.ledger_csv(serial, [(strategy, n, reports.peaks_by_category(worst))])
    hdr, rws = _rows(text)
    rhdr, rref = _rows(ref[f"ledger_n{n}_{strategy}"])
    assert hdr == rhdr
    assert [r[:3] for r in rws] == [r[:3] for r in rref]
    dup = {r[2]: int(r[4]) for r in rws if r[0] == strategy}
    assert dup["Param"] == 0 and dup["Grad"] == 0
