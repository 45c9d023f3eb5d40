"""The C-ABI library loads and exports every symbol include/skp.h declares;
the facade refuses to run without CUDA (no CPU fallback).  No compute calls."""
import os
import re

import pytest

from paper_2605_09755_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "skp.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skp_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.skp_abi_version() == 1


def test_ctypes_signatures_cover_header():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_exported_symbols_in_so():
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_no_cpu_fallback_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np
    import paper_2605_09755_b200 as skp
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        skp.make_sketch("countsketch", 10, 4, 0, s=2)
    spec = skp.RangeFinderSpec(k=2, l=4, r1=4, r2=3, q=1, eps=0.5, s=2)
    with pytest.raises(RuntimeError, match="CUDA"):
        skp.range_finder_sketched(np.ones((8, 6)), spec)


def test_spec_validation_messages():
    import paper_2605_09755_b200 as skp
    spec = skp.RangeFinderSpec(k=5, l=4, r1=10, r2=6, q=1, eps=0.5)
    with pytest.raises(ValueError, match="k <= l"):
        spec.validate(20, 20)
    with pytest.raises(ValueError, match="r2"):
        skp.RangeFinderSpec(k=3, l=4, r1=10, r2=2, q=1, eps=0.5).validate(20, 20)
    with pytest.raises(ValueError, match="eps"):
        skp.RangeFinderSpec(k=3, l=4, r1=10, r2=4, q=1, eps=0.7).validate(20, 20)
    assert skp.choose_q(0.5, 1) == 1
    assert skp.choose_q(0.1, 100) == 27


def test_sketch_space_rule_on_the_configs():
    """The power path each BASELINE config takes (CudaBackend.gram_ok's cost
    rule; profiles/r02w_c5_sweep.txt measured the C5 cases)."""
    from paper_2605_09755_b200._ops import gram_pays
    assert gram_pays(4000, 520, 3)            # C3: sketch space
    assert gram_pays(8000, 1050, 4)           # C5, the headline
    assert gram_pays(8000, 1050, 2)           # C5 q = 2 (was the products: 747 vs 699 ms)
    assert not gram_pays(8000, 1050, 1)       # C5 q = 1: three products are cheaper
    assert gram_pays(4000, 1050, 1)           # C5 l = 4000, q = 1
    assert not gram_pays(2000, 110, 3)        # C2: r2 small against l


def test_bench_arms_share_the_config():
    """Both bench arms print one config object (the driver compares them)."""
    import bench
    for name, cfg in bench.CONFIGS.items():
        a = bench.workload_config(name, cfg, 2)
        assert a == bench.workload_config(name, dict(cfg), 2)
        assert a["workload"] == name and "l2" in a and "parallelism" in a
