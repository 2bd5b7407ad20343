"""Trace files (workload.hpp:70-72, workload.cpp:108-137), CPU.

The replay input of bench_trace.py: workload.write_trace_csv / load_trace_csv must
produce and accept exactly the reference's format.  Pinned against the compiled
reference (dcpsim_ref::gen_trace + write_trace_csv / load_trace_csv):

* the CSV text of the same generated trace is byte-identical;
* loading the reference's CSV (also shuffled, with blank lines) gives the reference's
  own load_trace_csv result, ordered by (arrival, id);
* an empty file is a ConfigError in both.
"""
import ctypes
import random

import numpy as np
import pytest

from tests import oracle_lib
from paper_2605_21100_b200 import workload
from paper_2605_21100_b200._capi import ConfigError

P = oracle_lib.P


def _ref():
    L = oracle_lib.reference()
    if L is None:
        pytest.skip("oracle/_ref not built")
    L.dcpref_trace_csv.restype = ctypes.c_int64
    L.dcpref_trace_csv.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]
    L.dcpref_load_trace_csv.restype = ctypes.c_int
    L.dcpref_load_trace_csv.argtypes = [ctypes.c_char_p] + [ctypes.c_void_p] * 4 + [ctypes.c_int]
    return L


def _ref_csv(L, seed, long_ratio, rate, dur, poisson):
    n = L.dcpref_trace_csv(seed, long_ratio, rate, dur, poisson, None, 0)
    assert n >= 0
    buf = ctypes.create_string_buffer(n + 1)
    L.dcpref_trace_csv(seed, long_ratio, rate, dur, poisson, buf, n + 1)
    return buf.value.decode()


def _ref_load(L, text):
    cap = text.count("\n") + 1
    ids, arr = np.zeros(cap, np.int64), np.zeros(cap, np.float64)
    ln, out = np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    n = L.dcpref_load_trace_csv(text.encode(), P(ids), P(arr), P(ln), P(out), cap)
    if n < 0:
        return n
    return [(int(ids[i]), float(arr[i]), int(ln[i]), int(out[i])) for i in range(n)]


@pytest.mark.parametrize("seed,long_ratio,rate,dur,poisson", [
    (1, 0.01, 16.0, 20.0, 1), (7, 0.05, 64.0, 5.0, 1), (3, 0.0, 3.0, 10.0, 0), (42, 0.5, 9.7, 3.3, 0)])
def test_write_trace_csv_byte_identical(seed, long_ratio, rate, dur, poisson):
    L = _ref()
    tr = workload.gen_trace(seed, long_ratio, rate, dur, poisson=bool(poisson))
    assert workload.write_trace_csv(tr) == _ref_csv(L, seed, long_ratio, rate, dur, poisson)


def test_load_trace_csv_matches_reference():
    L = _ref()
    text = _ref_csv(L, 5, 0.05, 32.0, 8.0, 1)
    assert workload.load_trace_csv(text) == _ref_load(L, text)
    # out-of-order rows, duplicate arrivals and blank lines: both sort by (arrival, id)
    lines = text.strip().split("\n")
    body = lines[1:]
    random.Random(0).shuffle(body)
    body.insert(3, "")
    body.append("999,0.000,5,7")
    body.append("998,0.000,6,8")
    messy = "\n".join([lines[0]] + body) + "\n\n"
    got = workload.load_trace_csv(messy)
    assert got == _ref_load(L, messy)
    assert [r[0] for r in got[:2]] == [998, 999]  # poisson arrivals start after 0


def test_empty_trace_is_config_error():
    L = _ref()
    assert _ref_load(L, "") < 0
    with pytest.raises(ConfigError):
        workload.load_trace_csv("")


def test_round_trip_replays_same_requests():
    tr = workload.gen_trace(11, 0.01, 16.0, 5.0, poisson=True)
    back = workload.load_trace_csv(workload.write_trace_csv(tr))
    assert [(r[0], r[2], r[3]) for r in back] == [(r[0], r[2], r[3]) for r in tr]
    assert all(abs(a[1] - b[1]) <= 5e-4 for a, b in zip(back, tr))
