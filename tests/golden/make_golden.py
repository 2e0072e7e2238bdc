"""Generates tests/golden/bookkeeping.json from the REFERENCE ITSELF.

Loads oracle/_ref/libspecsim_ref.so — the reference's unmodified
perf_model.cpp / workload.cpp / rng.hpp compiled in place by
oracle/build_ref.sh — and records its outputs.  Run here (where
/root/reference exists):  make -C oracle ref && python tests/golden/make_golden.py
The committed JSON is what the GPU box and CPU tests compare against.
"""
import ctypes as C
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

R = oracle.ref()
SEEDS = [0, 7, 42, 12345, 20260217]
out = {"source": "oracle/_ref/libspecsim_ref.so built from /root/reference/proj/src "
                 "(perf_model.cpp, workload.cpp) + proj/include/specsim/rng.hpp"}

rng = {}
for s in SEEDS:
    h = R.ref_rng_create(s)
    uni = [R.ref_rng_uniform(h) for _ in range(32)]
    nor = [R.ref_rng_normal(h, 0.0, 1.0) for _ in range(16)]
    nor2 = [R.ref_rng_normal(h, 3.0, 2.0) for _ in range(8)]
    geo = {str(m): [R.ref_rng_geometric(h, m) for _ in range(16)] for m in (0.5, 1.0, 2.5, 100.0)}
    R.ref_rng_destroy(h)
    rng[str(s)] = dict(uniform=[x.hex() for x in uni], normal=[x.hex() for x in nor],
                       normal_3_2=[x.hex() for x in nor2], geometric=geo)
out["rng"] = rng

eal = []
for g in (1, 2, 3, 4, 5):
    for a in (0.0, 0.1, 0.25, 0.36, 0.5, 0.55, 0.6, 0.75, 0.9, 0.99, 1.0):
        o = C.c_double()
        assert R.ref_expected_accept_length(a, g, C.byref(o)) == 0
        eal.append([a, g, o.value.hex()])
out["expected_accept_length"] = eal

sal = []
for s, a, g in [(42, 0.6, 3), (7, 0.5, 3), (0, 0.0, 3), (1, 1.0, 3), (12345, 0.9, 5), (99, 0.3, 1)]:
    h = R.ref_rng_create(s)
    seq = []
    for _ in range(64):
        k = C.c_int()
        assert R.ref_sample_accept_length(h, a, g, C.byref(k)) == 0
        seq.append(k.value)
    R.ref_rng_destroy(h)
    sal.append(dict(seed=s, alpha=a, gamma=g, seq=seq))
out["sample_accept_length"] = sal

h = R.ref_rng_create(12345)
tot = 0
for _ in range(1_000_000):
    k = C.c_int()
    R.ref_sample_accept_length(h, 0.5, 3, C.byref(k))
    tot += k.value
R.ref_rng_destroy(h)
out["mc_mean_alpha0.5_gamma3_seed12345_1e6"] = tot / 1e6

afl = []
for g in (1, 3, 5):
    for ell in (1.0, 1.2, 1.47, 1.875, 2.0, 2.13, 2.5, 3.0, 3.9, g + 1.0):
        if ell > g + 1.0:
            continue
        o = C.c_double()
        assert R.ref_alpha_from_accept_length(ell, g, C.byref(o)) == 0
        afl.append([ell, g, o.value.hex()])
out["alpha_from_accept_length"] = afl

errs = []
o = C.c_double()
for a, g in [(-0.1, 3), (1.1, 3), (0.5, 0), (float("nan"), 3)]:
    errs.append(["expected_accept_length", a, g, R.ref_expected_accept_length(a, g, C.byref(o))])
for ell, g in [(0.9, 3), (4.5, 3), (2.0, 0)]:
    errs.append(["alpha_from_accept_length", ell, g, R.ref_alpha_from_accept_length(ell, g, C.byref(o))])
out["domain_errors"] = [[e[0], repr(e[1]), e[2], e[3]] for e in errs]

out["current_alpha"] = [[0.36, 0.55, 5000.0, n, R.ref_current_alpha(0.36, 0.55, 5000.0, n).hex()]
                        for n in (0.0, 1000.0, 5000.0, 20000.0)]
first = C.c_longlong()
tot = R.ref_workload_tokens(10, 100, 0.0, 7, C.byref(first))
out["workload_n10_mean100_seed7"] = dict(total=tot, first=first.value)

# SPEC known answers (not from code): SignalGeometry arithmetic
out["spec_bytes_100tok_h4096_3layers_bf16"] = 2457600
pathlib.Path(__file__).with_name("bookkeeping.json").write_text(json.dumps(out, indent=1))
print("wrote", pathlib.Path(__file__).with_name("bookkeeping.json"))
