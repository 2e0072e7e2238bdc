"""The C++ drop-in boundary coexists with the reference's own headers and
objects (VERDICT r1 "missing" #3).

A translation unit that includes the reference's errors.hpp, rng.hpp,
perf_model.hpp and workload.hpp (/root/reference/proj/include/specsim) and
this repo's proj/include/specsim/draft_trainer.hpp must compile, link against
the reference's perf_model.cpp / workload.cpp plus -lspecsim_draft, and run:
the reference's sample_accept_length and the library's C ABI give the same
draws, and a ConfigError thrown inside the library is caught as the
reference's specsim::ConfigError.  The library must export no symbol in
namespace specsim that the reference's objects define.

CPU only (the library loads without a GPU); skipped where the reference tree
is absent (the GPU box).
"""
import os
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF = pathlib.Path(os.environ.get("SPECSIM_REFERENCE", "/root/reference")) / "proj"
LIB = ROOT / "paper_2602_05145_b200" / "libspecsim_draft.so"

pytestmark = pytest.mark.skipif(not (REF / "src" / "perf_model.cpp").exists(),
                                reason="reference sources not present")

TU = r"""
#include "specsim/errors.hpp"
#include "specsim/rng.hpp"
#include "specsim/perf_model.hpp"
#include "specsim/workload.hpp"
#include "specsim/draft_trainer.hpp"
#include "specsim_draft_trainer.h"

#include <cstdio>
#include <stdexcept>

int main() {
  // the reference's own Rng and accept-length model (perf_model.cpp)...
  specsim::Rng ref_rng(20260217);
  specsim_rng* lib_rng = nullptr;
  if (specsim_rng_create(20260217, &lib_rng) != SPECSIM_OK) return 10;
  for (int i = 0; i < 1000; ++i) {
    const int a = specsim::sample_accept_length(ref_rng, 0.6, 3);
    int32_t b = 0;
    // ...and the library's restatement through the C ABI: same stream
    if (specsim_sample_accept_length(lib_rng, 0.6, 3, &b) != SPECSIM_OK) return 11;
    if (a != b) return 12;
  }
  specsim_rng_destroy(lib_rng);
  double lib_alpha = 0;
  specsim_alpha_from_accept_length(2.5, 3, &lib_alpha);
  if (lib_alpha != specsim::alpha_from_accept_length(2.5, 3)) return 13;
  // the reference's workload law next to the library's classes
  specsim::PhaseSpec ph;
  ph.alpha_start = 0.3;
  ph.alpha_ceiling = 0.8;
  ph.tau_samples = 100.0;
  if (!(specsim::current_alpha(ph, 50.0) > 0.3)) return 14;
  // ConfigError thrown inside the library == the reference's class
  int caught = 0;
  try {
    specsim::ControllerConfig c;
    c.lambda_short = 2.0;
    c.validate();
  } catch (const specsim::ConfigError& e) {
    caught = 1;
  }
  if (!caught) return 15;
  // domain errors stay std::invalid_argument (errors.hpp:8-9)
  caught = 0;
  try {
    specsim::SignalGeometry g;
    g.hidden_dim = 0;
    g.validate();
  } catch (const std::invalid_argument&) {
    caught = 1;
  }
  if (!caught) return 16;
  specsim::SignalGeometry g;
  g.hidden_dim = 4096;
  if (g.bytes_per_token() != 24576) return 17;  // SPEC.md:274
  std::puts("boundary ok");
  return 0;
}
"""


def _json_dir():
    import glob
    import sys
    p = glob.glob(sys.prefix + "/lib/python3*/site-packages/include/cudnn_frontend/thirdparty")
    return p[0] if p else None


def test_cpp_header_coexists_with_reference(tmp_path):
    assert LIB.exists(), "build the library first"
    src = tmp_path / "tu.cpp"
    src.write_text(TU)
    exe = tmp_path / "tu"
    jd = _json_dir()
    srcs = [str(src), str(REF / "src" / "perf_model.cpp")]
    incs = ["-I", str(REF / "include"), "-I", str(ROOT / "proj" / "include"),
            "-I", str(ROOT / "include")]
    if jd:
        srcs.append(str(REF / "src" / "workload.cpp"))
        incs += ["-I", jd, "-I", jd + "/nlohmann"]
    cmd = ["g++", "-std=c++20", "-Wall", "-Wextra", *incs, *srcs, "-o", str(exe),
           "-L", str(LIB.parent), "-lspecsim_draft", f"-Wl,-rpath,{LIB.parent}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "boundary ok" in out.stdout, (out.returncode, out.stderr)


def _defined(path, dynamic, strong_only=False):
    """Defined symbols; strong_only drops weak / COMDAT ones (W, V: inline
    members such as the shared ConfigError destructor are one definition by
    construction and merge at load time)."""
    args = ["nm", "-C", "--defined-only"] + (["-D"] if dynamic else []) + [str(path)]
    out = subprocess.run(args, capture_output=True, text=True, check=True).stdout
    kinds = "TDBR" if strong_only else "TDBRVW"
    syms = set()
    for line in out.splitlines():
        parts = line.split(" ", 2)
        if len(parts) == 3 and parts[1] in kinds:
            syms.add(parts[2])
    return syms


def test_library_exports_no_reference_symbol(tmp_path):
    objs = []
    jd = _json_dir()
    for name in ("perf_model.cpp", "workload.cpp") if jd else ("perf_model.cpp",):
        o = tmp_path / (name + ".o")
        subprocess.run(["g++", "-std=c++20", "-c", "-I", str(REF / "include"),
                        *(["-I", jd, "-I", jd + "/nlohmann"] if jd else []), str(REF / "src" / name), "-o", str(o)],
                       check=True)
        objs.append(o)
    ref = set()
    for o in objs:
        ref |= {s for s in _defined(o, False, strong_only=True) if s.startswith("specsim::")}
    assert any("sample_accept_length" in s for s in ref)
    exported = {s for s in _defined(LIB, True) if s.startswith("specsim::")}
    clash = sorted(ref & exported)
    assert not clash, clash
    # the bookkeeping restatement stays internal (hidden visibility)
    assert not any(("accept_length" in s or "Rng::" in s) for s in exported), sorted(exported)[:20]
