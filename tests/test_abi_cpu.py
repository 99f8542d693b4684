"""CPU: the C-ABI library loads without a GPU, exports every symbol include/regot_b200.h declares,
the ctypes struct layouts match the C ones, and compute entry points fail loudly with no device."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

import paper_2605_08793_b200 as rg
from paper_2605_08793_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "regot_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(regot_b200_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    names = declared_symbols()
    assert len(names) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (regot_b200_\w+)", out))
    assert set(names) <= exported, sorted(set(names) - exported)
    assert set(names) == set(_lib.PROTOTYPES), sorted(set(names) ^ set(_lib.PROTOTYPES))
    lib = _lib.load()
    assert lib.regot_b200_version().decode().startswith("regot_b200") and b"sm_100a" in lib.regot_b200_version()


def test_library_contains_only_sm100a_code():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_ctypes_struct_layouts_match_c():
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "regot_b200.h"
#define P(t, f) printf(#t "." #f " %zu\n", offsetof(t, f))
int main(void) {
  printf("regot_splr_config %zu\n", sizeof(regot_splr_config));
  P(regot_splr_config, overlap); P(regot_splr_config, cg_max_iter); P(regot_splr_config, cg_rtol);
  printf("regot_sinkhorn_config %zu\n", sizeof(regot_sinkhorn_config));
  printf("regot_trace_row %zu\n", sizeof(regot_trace_row));
  printf("regot_step_record %zu\n", sizeof(regot_step_record));
  P(regot_step_record, curvature_ok); P(regot_step_record, tau); P(regot_step_record, cg_iters);
  printf("regot_result %zu\n", sizeof(regot_result));
  P(regot_result, trace); P(regot_result, eta); P(regot_result, algo); P(regot_result, message); P(regot_result, device_ms);
  P(regot_result, kernel_launches);
  printf("regot_gradient_info %zu\n", sizeof(regot_gradient_info));
  return 0; }
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "layout.c")
        open(src, "w").write(prog)
        exe = os.path.join(d, "layout")
        subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), "-o", exe, src], check=True)  # header is plain C
        got = dict(line.rsplit(" ", 1) for line in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines())
    want = {
        "regot_splr_config": C.sizeof(_lib.SplrConfigC),
        "regot_splr_config.overlap": _lib.SplrConfigC.overlap.offset,
        "regot_splr_config.cg_max_iter": _lib.SplrConfigC.cg_max_iter.offset,
        "regot_splr_config.cg_rtol": _lib.SplrConfigC.cg_rtol.offset,
        "regot_sinkhorn_config": C.sizeof(_lib.SinkhornConfigC),
        "regot_trace_row": C.sizeof(_lib.TraceRowC),
        "regot_step_record": C.sizeof(_lib.StepRecordC),
        "regot_step_record.curvature_ok": _lib.StepRecordC.curvature_ok.offset,
        "regot_step_record.tau": _lib.StepRecordC.tau.offset,
        "regot_step_record.cg_iters": _lib.StepRecordC.cg_iters.offset,
        "regot_result": C.sizeof(_lib.ResultC),
        "regot_result.trace": _lib.ResultC.trace.offset,
        "regot_result.eta": _lib.ResultC.eta.offset,
        "regot_result.algo": _lib.ResultC.algo.offset,
        "regot_result.message": _lib.ResultC.message.offset,
        "regot_result.device_ms": _lib.ResultC.device_ms.offset,
        "regot_result.kernel_launches": _lib.ResultC.kernel_launches.offset,
        "regot_gradient_info": C.sizeof(_lib.GradientInfoC),
    }
    assert {k: int(v) for k, v in got.items()} == want


def test_cxx_shim_compiles_against_the_abi():
    # include/regot_b200.hpp re-creates regot::run_splr-shaped wrappers; compile and link (no run: no GPU here)
    prog = r'''
#include "regot_b200.hpp"
int main() {
  regot_b200::ProblemInstance p; p.n = 2; p.m = 2; p.M = {0, 0, 0, 0}; p.a = {.5, .5}; p.b = {.5, .5}; p.eta = 1.0;
  try {
    regot_b200::Solver s(0);
    s.set_problem(p);
    regot_b200::SplrConfig cfg;
    regot_b200::SplrResult r = s.run_splr(regot_b200::DualPoint::zeros(2, 2), cfg);
    return r.trace.rows.empty();
  } catch (const regot_b200::Error& e) { return 42; }
}
'''
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "shim.cpp")
        open(src, "w").write(prog)
        exe = os.path.join(d, "shim")
        libdir = os.path.dirname(_lib.LIB_PATH)
        subprocess.run(["g++", "-std=c++17", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", exe, src, "-L", libdir,
                        "-lregot_b200", f"-Wl,-rpath,{libdir}", "-L/usr/local/cuda/lib64", "-Wl,-rpath,/usr/local/cuda/lib64"], check=True)
        import torch
        if not torch.cuda.is_available():
            # without a device the shim must surface the library's loud failure as an exception
            assert subprocess.run([exe]).returncode == 42


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rg.CudaError, match="no CPU fallback"):
        rg.Solver(0)


def test_status_names_mirror_reference_exception_classes():
    lib = _lib.load()
    names = {1: "DegenerateCostError", 2: "FormatError", 3: "TruncationError", 4: "ValidationError", 5: "IoError",
             6: "OracleSizeError", 7: "StructureError", 8: "NotPositiveDefiniteError", 9: "DirectionError",
             10: "LineSearchError", 11: "PlotError", 12: "StepError"}
    for code, nm in names.items():
        assert lib.regot_b200_status_name(code).decode() == nm
        assert rg.regot._ERRORS.get(code, rg.StepError).__name__ == nm
