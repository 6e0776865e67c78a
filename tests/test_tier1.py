"""Tier-1 ingestion (SPEC S:45-79 interface): canonical
CSV -> records -> schema -> the lattice arrays of sr_load_dataset.  CPU only."""
import numpy as np
import pytest

import gen
from paper_1910_07776_b200 import tier1 as T

HDR = "program,input_id,run_id,version_mask,kernel,counter,value\n"


def test_spec_three_row_group():
    # {inst_executed=500, elapsed_cycles=1000, runtime_ms=2.5} -> one record
    recs = T.parse_canonical_csv(HDR + "BH,in0,0,0,k,inst_executed,500\nBH,in0,0,0,k,elapsed_cycles,1000\n"
                                       "BH,in0,0,0,k,runtime_ms,2.5\n")
    assert len(recs) == 1
    r = recs[0]
    assert r.counters == {"inst_executed": 500.0} and r.cycles == 1000.0 and r.runtime == 2.5


def test_spec_empty_and_two_runs_and_comments():
    assert T.parse_canonical_csv(HDR) == []
    text = HDR + "# comment\n" + "".join(
        f"P,i,{run},0,k,{c},{v}\n" for run in (0, 1) for c, v in (("x", 1), ("elapsed_cycles", 10), ("runtime_ms", 1)))
    recs = T.parse_canonical_csv(text)
    assert len(recs) == 2 and {r.run_id for r in recs} == {0, 1}
    assert len({r.key for r in recs}) == 2


@pytest.mark.parametrize("text, msg", [
    (HDR + "P,i,0,0,k,x\n", "line 2"),                                    # wrong column count
    (HDR + "P,i,zero,0,k,x,1\n", "line 2"),                               # non-numeric
    (HDR + "P,i,0,0,k,x,1\nP,i,0,0,k,x,2\n", "duplicate"),               # duplicate counter
    (HDR + "P,i,0,0,k,x,1\nP,i,0,0,k,runtime_ms,1\n", "incomplete"),     # missing cycles
    (HDR + "P,i,0,0,k,x,-1\nP,i,0,0,k,elapsed_cycles,1\nP,i,0,0,k,runtime_ms,1\n", "negative"),
    (HDR + "P,i,0,0,k,elapsed_cycles,0\nP,i,0,0,k,runtime_ms,1\n", "> 0"),
])
def test_parse_errors_name_the_problem(text, msg):
    with pytest.raises(T.Tier1Error, match=msg):
        T.parse_canonical_csv(text)


def test_schema_intersection_examples():
    R = T.Record
    assert T.build_schema([R("p", "i", 0, 0, "k", {"a": 1, "b": 1, "c": 1}), R("p", "i", 1, 0, "k", {"b": 1, "c": 1, "d": 1})]) == ["b", "c"]
    assert T.build_schema([R("p", "i", 0, 0, "k", {"a": 1})]) == ["a"]
    with pytest.raises(T.Tier1Error, match="share no counter"):
        T.build_schema([R("p", "i", 0, 0, "k", {"a": 1}), R("p", "i", 1, 0, "k", {"b": 1})])


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_round_trip_reproduces_the_lattice(name):
    """gen dataset -> canonical CSV -> parse -> to_dataset reproduces every
    array exactly (counters, cycles, runtimes, opt bits), and
    parse(serialize(records)) == records."""
    ds = gen.make_config(name).dataset
    recs = T.dataset_to_records(ds)
    text = T.serialize_canonical_csv(recs)
    back = T.parse_canonical_csv(text)
    assert [(r.key, r.counters, r.cycles, r.runtime) for r in back] == \
           [(r.key, r.counters, r.cycles, r.runtime) for r in recs]
    ds2, info = T.to_dataset(back)
    assert (ds2.n_programs, ds2.n_inputs, ds2.n_runs, ds2.n_opt_bits, ds2.n_counters) == \
           (ds.n_programs, ds.n_inputs, ds.n_runs, ds.n_opt_bits, ds.n_counters)
    assert np.array_equal(ds2.opt_bit[:, :ds.n_opt_ids], ds.opt_bit)
    for f in ("counters", "cycles", "runtime_ms"):
        assert np.array_equal(getattr(ds2, f), getattr(ds, f)), f


def test_lattice_errors():
    ds = gen.make_config("C1").dataset
    recs = T.dataset_to_records(ds)
    with pytest.raises(T.Tier1Error, match="missing version"):
        T.to_dataset(recs[:-1])
    with pytest.raises(T.Tier1Error, match="duplicate"):
        T.to_dataset(recs + [recs[0]])
    other = [T.Record("Q", r.input_id, r.run_id, r.version_mask & 0b111, r.kernel, r.counters, r.cycles, r.runtime)
             for r in recs if r.version_mask < 8]
    with pytest.raises(T.Tier1Error, match="optimizations"):
        T.to_dataset(recs + other)


NVPROF = """==PROF== Connected to process 1234
==1234== Profiling application: ./bh 500000 10
==1234== Event result:
"Device","Kernel","Invocations","Event Name","Min","Max","Avg","Total"
"Tesla K20c (0)","ForceCalculationKernel","10","inst_executed","900","1100","1000","10000"
"Tesla K20c (0)","ForceCalculationKernel","10","elapsed_cycles_sm","1900","2100","2000","20000"
"Tesla K20c (0)","SortKernel","10","inst_executed","40","60","50","500"
"""


def test_nvprof_import_spec_examples():
    # Device,Kernel,Event Name,Min,Max,Avg -> the event's Avg value; "==" lines skipped
    recs = T.import_nvprof_csv(NVPROF, "BH", "in5", 0, 0b1011, runtime_ms=2.5, kernel="ForceCalculationKernel")
    assert len(recs) == 1
    r = recs[0]
    assert r.counters == {"inst_executed": 1000.0} and r.cycles == 2000.0 and r.runtime == 2.5
    assert r.key == ("BH", "in5", 0, 0b1011, "ForceCalculationKernel")
    # an export lacking the cycles event -> incomplete-record error
    with pytest.raises(T.Tier1Error, match="incomplete"):
        T.import_nvprof_csv(NVPROF, "BH", "in5", 0, 0, runtime_ms=1.0, kernel="SortKernel")
    with pytest.raises(T.Tier1Error, match="header"):
        T.import_nvprof_csv("==PROF== nothing\n1,2,3\n", "BH", "i", 0, 0)
