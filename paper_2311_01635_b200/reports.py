"""The reference's memory reports from the DEVICE ledger:
`rtpsim memtable`, `rtpsim ledger` and `rtpsim sweep` CSVs
(proj/src/commands.cpp:87-181) with the same headers, column order, row order
and strategy / category names, the byte columns filled from the per-worker
device ledgers of an RTP run (bf16 weights, fp32 gradients) instead of the
reference's fp64 simulation. The analytic Table-1 rows
(analysis.cpp:32-49, `table1_memory`) are restated for the memtable report.
"""
from __future__ import annotations

MEMTABLE_HEADER = "strategy,n,activation_mem,param_mem,duplication"
LEDGER_HEADER = "strategy,n,category,peak_bytes,duplication"
SWEEP_HEADER = ("strategy,n,batch_per_worker,global_batch,param_peak,grad_peak,activation_peak,"
                "commbuffer_peak,other_peak,total_peak")
# analysis.cpp:11-22 order (kAllStrategies) and names
STRATEGIES = ("no-parallelism", "tensor-parallel", "data-parallel", "pipeline-parallel", "fsdp", "rtp",
              "rtp-inplace")
# ledger.cpp mem_category_name order
CATEGORIES = ("Param", "Grad", "Activation", "CommBuffer", "Other")
_KEYS = ("param", "grad", "activation", "comm", "other")


def table1_memory(strategy: str, W: int, G: int, A: int, Ap: int, N: int) -> tuple[int, int, int]:
    """(activation_mem, param_mem, duplication): whole-system bytes of the
    paper's Table 1 (analysis.cpp:32-49)."""
    if N == 0:
        raise ValueError("table1_memory: N must be >= 1")
    if N == 1:
        return A, W + G, 0
    mx = max(W, G)
    return {
        "no-parallelism": (A, W + G, 0),
        "tensor-parallel": (A * N, W + G, A * (N - 1)),
        "data-parallel": (A, (W + G) * N, (W + G) * (N - 1)),
        "pipeline-parallel": (A + Ap * N, W + G, Ap * N),
        "fsdp": (A, W + G + mx * (N - 1), mx * (N - 1)),
        "rtp": (A, W + G + mx, mx),
        "rtp-inplace": (A, W + G, 0),
    }[strategy]


def memtable_csv(N: int, W: int, G: int, A: int, Ap: int) -> str:
    """`rtpsim memtable` (commands.cpp:87-110): the seven analytic rows."""
    lines = [MEMTABLE_HEADER]
    for s in STRATEGIES:
        a, p, d = table1_memory(s, W, G, A, Ap, N)
        lines.append(f"{s},{N},{a},{p},{d}")
    return "\n".join(lines) + "\n"


def device_memtable_rows(N: int, W: int, G: int, ledgers_inplace, ledgers_outofplace) -> str:
    """The two RTP rows of Table 1 MEASURED: whole-system activation and
    Param+Grad+CommBuffer peaks summed over the N workers' device ledgers
    (rtpb_group_ledger dicts), duplication against the serial W + G."""
    lines = [MEMTABLE_HEADER]
    for name, leds in (("rtp", ledgers_outofplace), ("rtp-inplace", ledgers_inplace)):
        act = sum(d["peak_activation"] for d in leds)
        pgc = sum(d["peak_param"] + d["peak_grad"] + d["peak_comm"] for d in leds)
        lines.append(f"{name},{N},{act},{pgc},{pgc - (W + G)}")
    return "\n".join(lines) + "\n"


def peaks_by_category(ledger: dict) -> dict:
    """rtpb_group_ledger dict -> {category name: peak bytes}."""
    return {c: int(ledger["peak_" + k]) for c, k in zip(CATEGORIES, _KEYS)}


def ledger_csv(serial: dict, runs) -> str:
    """`rtpsim ledger` (commands.cpp:112-143). serial: category peaks of the
    one-worker run; runs: [(strategy name, n, category peaks of the worst
    worker)], serial listed first as the reference does. duplication =
    n * peak - serial peak (analysis.cpp:335-340)."""
    lines = [LEDGER_HEADER]
    for name, n, pk in [("serial", 1, serial)] + list(runs):
        for c in CATEGORIES:
            lines.append(f"{name},{n},{c},{pk[c]},{n * pk[c] - serial[c]}")
    return "\n".join(lines) + "\n"


def sweep_csv(strategy: str, n: int, points) -> str:
    """`rtpsim sweep` (commands.cpp:165-181). points: [(batch_per_worker,
    category peaks, total peak)]."""
    lines = [SWEEP_HEADER]
    for b, pk, total in points:
        lines.append(f"{strategy},{n},{b},{b * n},{pk['Param']},{pk['Grad']},{pk['Activation']},"
                     f"{pk['CommBuffer']},{pk['Other']},{total}")
    return "\n".join(lines) + "\n"
