"""Host logic of bench.py's roofline objects (no GPU): the composite V-cycle roofline, its directly
timed / profiled / in-solve fractions, and the binding-bound choice of a tensor-class kernel below the
ridge."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("rte_bench", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)

PEAKS = {"hbm_gbs": 6500.0, "bf16_tflops": 1650.0, "bf16_tflops_sustained": 1380.0, "sm_max_mhz": 1965.0}


def _classes():
    # 10 V-cycles: a tensor-bound conv class, an HBM-bound 1x1 class (once per V-cycle), and one Arnoldi class
    return [
        {"name": "conv3x3_tc@512x32->32", "kind": "tensor_3xtf32", "launches": 80, "ms": 4.0,
         "flops": 80 * 4.8e9, "bytes": 80 * 1.0e8},
        {"name": "conv1x1_tc@512x256->32", "kind": "tensor_3xtf32", "launches": 10, "ms": 0.7,
         "flops": 10 * 4.3e9, "bytes": 10 * 3.0e8},
        {"name": "dcgs_update", "kind": "hbm", "launches": 10, "ms": 8.0, "flops": 0.0, "bytes": 10 * 5.0e9},
    ]


def test_composite_vcycle_roofline_and_its_three_timings():
    cl = _classes()
    rv = bench._composite_roofline(cl, lambda n: not n.startswith(bench._NOT_VCYCLE), PEAKS, "V")
    burst, sus = bench._tensor_peaks(PEAKS)
    t_conv = 80 * 4.8e9 / (burst * 1e12) * 1e3            # tensor-bound
    t_lift = 10 * 3.0e8 / (PEAKS["hbm_gbs"] * 1e9) * 1e3  # HBM-bound although a tensor-class kernel
    assert abs(rv["roofline_ms_burst"] - (t_conv + t_lift)) < 1e-9
    assert abs(rv["frac"] - (t_conv + t_lift) / 4.7) < 1e-12
    rv = bench._vcycle_direct(rv, cl, {"mgnet_vcycle_per_s": 1e3 / 0.40}, timed_ms=13.0)
    assert rv["vcycles_profiled"] == 10
    assert abs(rv["frac_profiled"] - (t_conv + t_lift) / 4.7) < 1e-12
    assert abs(rv["frac"] - (t_conv + t_lift) / 10 / 0.40) < 1e-12
    # in-solve bound: (13.0 - 8.0) / 10 V-cycles = 0.5 ms
    assert abs(rv["in_solve"]["ms_per_vcycle_upper_bound"] - 0.5) < 1e-12
    assert rv["in_solve"]["frac"] < rv["frac"] and rv["frac_sustained"] > rv["frac"]


def test_tensor_class_below_the_ridge_reports_the_hbm_bound():
    cl = _classes()
    roof, _ = bench._roofline(cl, PEAKS, "test", top=cl[1])
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert abs(roof["achieved"] - 3.0e8 / (0.07e-3) / 1e9) < 1e-6
    roof, _ = bench._roofline(cl, PEAKS, "test", top=cl[0])
    assert roof["bound"] == "tensor" and "frac_sustained" in roof
