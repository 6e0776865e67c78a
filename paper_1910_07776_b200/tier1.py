"""Tier-1 ingestion: profiler counters in the canonical
CSV interchange format -> the lattice arrays `sr_load_dataset` takes.

The paper's Tier 1 "profiles the user's code ... measures a large number of
hardware performance counter events" and normalises them by cycles;
the counters of every version of the 2^m optimization lattice are what the
GPU path consumes.  This module is the host-side plumbing in front of it:

    parse_canonical_csv(text) -> [Record]        (SPEC S:45-55 interface)
    serialize_canonical_csv(records) -> text     (round trip)
    build_schema(records) -> [counter names]     (sorted intersection)
    to_dataset(records, kernel=None) -> Dataset   (the sr_dataset lattice)

Canonical format (one value per row, `#` comments):
    program,input_id,run_id,version_mask,kernel,counter,value
`version_mask` bit i set = optimization id i applied; the counters
`elapsed_cycles` (integer) and `runtime_ms` (real) are the normaliser and
the runtime, not features.  Errors are `Tier1Error` naming the line or the
offending (program, input, run, version).  Parsing is host work by nature
(text in, arrays out); nothing of the Tier-2/3 computation happens here.
"""
from __future__ import annotations

import csv
import io
import math
from dataclasses import dataclass, field

import numpy as np

RESERVED = ("elapsed_cycles", "runtime_ms")
HEADER = ["program", "input_id", "run_id", "version_mask", "kernel", "counter", "value"]


class Tier1Error(ValueError):
    """Malformed, incomplete or inconsistent Tier-1 input (message names the line or group)."""


@dataclass
class Record:
    program: str
    input_id: str
    run_id: int
    version_mask: int
    kernel: str
    counters: dict = field(default_factory=dict)
    cycles: float = float("nan")
    runtime: float = float("nan")

    @property
    def key(self):
        return (self.program, self.input_id, self.run_id, self.version_mask, self.kernel)


def parse_canonical_csv(text: str) -> list:
    """One Record per (program, input_id, run_id, version_mask, kernel) group, in
    first-appearance order.  Errors: wrong column count / non-numeric value
    (line number), duplicate (group, counter), missing elapsed_cycles or
    runtime_ms (group named), non-positive cycles / runtime, negative count."""
    recs: dict = {}
    seen_header = False
    for ln, row in enumerate(csv.reader(io.StringIO(text)), start=1):
        if not row or (row[0].strip().startswith("#")):
            continue
        row = [c.strip() for c in row]
        if not seen_header and row == HEADER:
            seen_header = True
            continue
        if len(row) != 7:
            raise Tier1Error(f"line {ln}: expected 7 columns, got {len(row)}")
        prog, inp, run, mask, kern, name, val = row
        try:
            run_i, mask_i, v = int(run), int(mask), float(val)
        except ValueError:
            raise Tier1Error(f"line {ln}: non-numeric run_id / version_mask / value") from None
        if run_i < 0 or mask_i < 0:
            raise Tier1Error(f"line {ln}: run_id and version_mask must be >= 0")
        if not math.isfinite(v):
            raise Tier1Error(f"line {ln}: non-finite value")
        key = (prog, inp, run_i, mask_i, kern)
        r = recs.get(key)
        if r is None:
            r = recs[key] = Record(prog, inp, run_i, mask_i, kern)
        if name == "elapsed_cycles":
            if not math.isnan(r.cycles):
                raise Tier1Error(f"line {ln}: duplicate elapsed_cycles for {key}")
            r.cycles = v
        elif name == "runtime_ms":
            if not math.isnan(r.runtime):
                raise Tier1Error(f"line {ln}: duplicate runtime_ms for {key}")
            r.runtime = v
        else:
            if name in r.counters:
                raise Tier1Error(f"line {ln}: duplicate counter {name!r} for {key}")
            if v < 0:
                raise Tier1Error(f"line {ln}: negative count for {name!r}")
            r.counters[name] = v
    out = list(recs.values())
    for r in out:
        if math.isnan(r.cycles) or math.isnan(r.runtime):
            raise Tier1Error(f"incomplete record {r.key}: missing elapsed_cycles or runtime_ms")
        if not (r.cycles > 0 and r.runtime > 0):
            raise Tier1Error(f"record {r.key}: elapsed_cycles and runtime_ms must be > 0")
    return out


def import_nvprof_csv(text: str, program: str, input_id: str, run_id: int, version_mask: int,
                      runtime_ms: float | None = None, kernel: str | None = None,
                      cycles_event: str = "elapsed_cycles_sm") -> list:
    """Best-effort import of an nvprof event / metric CSV export (SPEC S:56-63,
    P:175 "nvprof from the Visual Profiler"): `==` comment lines skipped; a
    header row with a "Kernel" column and a value column (Avg preferred, else
    Value / Max); one Record per kernel with the caller's identity labels.
    `cycles_event` names the cycle counter (stored as elapsed_cycles); the
    runtime comes from `runtime_ms` (nvprof's event export has none).
    Errors: no recognizable header -> Tier1Error; missing cycles -> incomplete."""
    rows = [r for r in csv.reader(io.StringIO(text)) if r and not r[0].lstrip().startswith("==")]
    hdr_i = next((i for i, r in enumerate(rows) if any(c.strip() == "Kernel" for c in r)), None)
    if hdr_i is None:
        raise Tier1Error("nvprof: no header row with a Kernel column")
    hdr = [c.strip() for c in rows[hdr_i]]
    k_col = hdr.index("Kernel")
    n_col = next((hdr.index(h) for h in ("Event Name", "Metric Name") if h in hdr), None)
    v_col = next((hdr.index(h) for h in ("Avg", "Value", "Max") if h in hdr), None)
    if n_col is None or v_col is None:
        raise Tier1Error("nvprof: header lacks an event/metric name or value column")
    recs: dict = {}
    for ln, r in enumerate(rows[hdr_i + 1:], start=hdr_i + 2):
        if len(r) <= max(k_col, n_col, v_col):
            continue
        kern = r[k_col].strip()
        if kernel is not None and kern != kernel:
            continue
        name, val = r[n_col].strip(), r[v_col].strip().rstrip("%")
        try:
            v = float(val)
        except ValueError:
            raise Tier1Error(f"nvprof line {ln}: non-numeric value {val!r}") from None
        rec = recs.setdefault(kern, Record(program, input_id, int(run_id), int(version_mask), kern))
        if name == cycles_event:
            rec.cycles = v
        else:
            rec.counters[name] = v
    out = list(recs.values())
    for r in out:
        if runtime_ms is not None:
            r.runtime = float(runtime_ms)
        if math.isnan(r.cycles):
            raise Tier1Error(f"incomplete record {r.key}: no {cycles_event} event")
    return out


def serialize_canonical_csv(records) -> str:
    """Canonical CSV of the records (counters in name order, then the two
    reserved rows); repr() floats, so parse(serialize(r)) == r exactly."""
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(HEADER)
    for r in records:
        base = [r.program, r.input_id, r.run_id, r.version_mask, r.kernel]
        for name in sorted(r.counters):
            w.writerow(base + [name, repr(float(r.counters[name]))])
        w.writerow(base + ["elapsed_cycles", repr(float(r.cycles))])
        w.writerow(base + ["runtime_ms", repr(float(r.runtime))])
    return buf.getvalue()


def build_schema(records) -> list:
    """Counter names common to every record, sorted (deterministic in record order)."""
    if not records:
        raise Tier1Error("schema: no records")
    common = set(records[0].counters)
    for r in records[1:]:
        common &= set(r.counters)
    if not common:
        raise Tier1Error("schema: the records share no counter")
    return sorted(common)


def to_dataset(records, schema=None, kernel=None, opt_names=None):
    """Assemble the version lattice sr_load_dataset takes (gen.synth.Dataset).

    Programs, inputs and runs are taken in sorted order; program p's lattice
    bits are its optimization ids (bits present in its version masks) in
    ascending order, so `opt_bit[p][o]` = rank of id o among them (-1 if p
    never applies o) and version v of the lattice is the mask compressed onto
    those bits.  Every (program, input, run) group must hold all 2^m versions,
    every program the same m and the same number of inputs and runs (the
    slot layout t = ((p*I + i)*R + r)*2^m + v).  Returns (dataset, info) with
    the label maps in `info`."""
    from gen.synth import Dataset
    recs = [r for r in records if kernel is None or r.kernel == kernel]
    if not recs:
        raise Tier1Error(f"no records for kernel {kernel!r}")
    kernels = {r.kernel for r in recs}
    if len(kernels) > 1:
        raise Tier1Error(f"records of several kernels {sorted(kernels)}: pass kernel=")
    schema = schema or build_schema(recs)
    progs = sorted({r.program for r in recs})
    ids_of = {p: sorted({b for r in recs if r.program == p for b in range(r.version_mask.bit_length())
                         if (r.version_mask >> b) & 1}) for p in progs}
    m = len(ids_of[progs[0]])
    for p in progs:
        if len(ids_of[p]) != m:
            raise Tier1Error(f"program {p!r} has {len(ids_of[p])} optimizations, {progs[0]!r} has {m}")
    inputs = {p: sorted({r.input_id for r in recs if r.program == p}) for p in progs}
    runs = {p: sorted({r.run_id for r in recs if r.program == p}) for p in progs}
    I, R = len(inputs[progs[0]]), len(runs[progs[0]])
    for p in progs:
        if len(inputs[p]) != I or len(runs[p]) != R:
            raise Tier1Error(f"program {p!r}: {len(inputs[p])} inputs x {len(runs[p])} runs, expected {I} x {R}")
    n_ids = max((max(v) + 1 if v else 0) for v in ids_of.values())
    O = max(n_ids, 1)
    P, V, C = len(progs), 1 << m, len(schema)
    N = P * I * R * V
    opt_bit = np.full((P, O), -1, dtype=np.int8)
    for pi, p in enumerate(progs):
        for b, oid in enumerate(ids_of[p]):
            opt_bit[pi, oid] = b
    counters = np.zeros((N, C))
    cycles = np.zeros(N)
    runtime = np.zeros(N)
    filled = np.zeros(N, dtype=bool)
    index = {p: (pi, {x: k for k, x in enumerate(inputs[p])}, {x: k for k, x in enumerate(runs[p])})
             for pi, p in enumerate(progs)}
    for r in recs:
        pi, imap, rmap = index[r.program]
        ids = ids_of[r.program]
        if r.version_mask & ~sum(1 << i for i in ids):
            raise Tier1Error(f"record {r.key}: version_mask uses an optimization id the program lacks")
        v = sum(1 << b for b, oid in enumerate(ids) if (r.version_mask >> oid) & 1)
        t = ((pi * I + imap[r.input_id]) * R + rmap[r.run_id]) * V + v
        if filled[t]:
            raise Tier1Error(f"duplicate record {r.key}")
        try:
            counters[t] = [r.counters[n] for n in schema]
        except KeyError as e:
            raise Tier1Error(f"record {r.key}: missing counter {e.args[0]!r}") from None
        cycles[t], runtime[t], filled[t] = r.cycles, r.runtime, True
    if not filled.all():
        t = int(np.argmin(filled))
        v, g = t % V, t // V
        p, rest = divmod(g, I * R)
        i, rr = divmod(rest, R)
        mask = sum(1 << oid for b, oid in enumerate(ids_of[progs[p]]) if (v >> b) & 1)
        raise Tier1Error(f"missing version: program {progs[p]!r} input {inputs[progs[p]][i]!r} "
                         f"run {runs[progs[p]][rr]} version_mask {mask}")
    ds = Dataset(n_programs=P, n_inputs=I, n_runs=R, n_opt_bits=m, n_counters=C, n_opt_ids=O,
                 counters=counters, cycles=cycles, runtime_ms=runtime, opt_bit=opt_bit,
                 opt_names=list(opt_names) if opt_names else [f"opt{o}" for o in range(O)],
                 program_names=progs)
    info = {"schema": schema, "programs": progs, "inputs": inputs, "runs": runs, "opt_ids": ids_of}
    return ds, info


def dataset_to_records(ds, kernel: str = "kernel", input_names=None) -> list:
    """The inverse of to_dataset for a lattice whose program p applies ids with
    opt_bit[p] >= 0 (used to export synthetic datasets in the canonical form)."""
    P, I, R, m, C = ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_opt_bits, ds.n_counters
    V = 1 << m
    names = [f"c{c:03d}" for c in range(C)]
    progs = list(ds.program_names) if ds.program_names else [f"p{p}" for p in range(P)]
    out = []
    for p in range(P):
        bit_to_id = {int(b): o for o, b in enumerate(ds.opt_bit[p]) if b >= 0}
        for i in range(I):
            for r in range(R):
                for v in range(V):
                    t = ((p * I + i) * R + r) * V + v
                    mask = sum(1 << bit_to_id[b] for b in range(m) if (v >> b) & 1)
                    rec = Record(progs[p], (input_names or {}).get(i, f"in{i}"), r, mask, kernel,
                                 {names[c]: float(ds.counters[t, c]) for c in range(C)},
                                 float(ds.cycles[t]), float(ds.runtime_ms[t]))
                    out.append(rec)
    return out
