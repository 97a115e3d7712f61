"""CPU-side checks of the boundary: the C-ABI library loads without a GPU and exports every symbol that
include/hisa_cuda.h declares; config validation (pure host logic) behaves like the reference constructor."""
import json
import os
import re

import pytest

from paper_2603_28458_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    capi.build()
    return capi.lib()


def test_header_symbols_are_all_exported(lib):
    header = open(os.path.join(ROOT, "include", "hisa_cuda.h")).read()
    declared = sorted(set(re.findall(r"\b(hisa_cuda_[a-z_0-9]+)\s*\(", header)))
    assert declared, "no declarations found"
    assert sorted(capi.EXPORTED_SYMBOLS) == declared
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in hisa_cuda.h but not exported"


def test_abi_version_and_status_names(lib):
    assert lib.hisa_cuda_abi_version() == 1
    assert lib.hisa_cuda_status_name(1) == b"InfeasibleConfig"
    assert lib.hisa_cuda_status_name(3) == b"EmptySequence"
    assert lib.hisa_cuda_status_name(10) == b"NoDevice"


def test_config_validation_matches_reference_ctor(lib):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "ref_golden.json")))
    for B, m, k, H, d, ok in gold["config_cases"]:
        cfg = capi.make_config(B, m, k, H, d)
        if ok:
            capi.config_validate(cfg)
        else:
            with pytest.raises(capi.HisaError) as e:
                capi.config_validate(cfg)
            assert e.value.name == "InfeasibleConfig"
    cfg = capi.make_config(128, 64, 2048, 64, 128)
    g = gold["config_defaults"]
    assert (cfg.force_first_last, cfg.forced_in_budget, cfg.tie_break, cfg.pool_mode) == (
        g["force_first_last"], g["forced_in_budget"], g["tie_break"], g["pool_mode"])


def test_no_cpu_fallback_without_device(lib):
    if capi.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(capi.HisaError) as e:
        capi.Indexer(capi.make_config())
    assert e.value.name == "NoDevice"


def test_bf16_rounding_helpers():
    import numpy as np
    x = np.float32([1.0, 1.00390625, 1.0078125, -3.14159, 1e-40, 65504.0])
    b = capi.f32_to_bf16_bits(x)
    back = capi.bf16_bits_to_f32(b)
    assert back[0] == 1.0 and back[1] == 1.0 and back[2] == 1.0078125  # ties-to-even at 1 + 2^-8
    assert np.all(np.abs(back[3] - x[3]) <= 2 ** -7 * abs(x[3]))


def test_e4m3_helpers_round_trip_and_rounding():
    import numpy as np
    allb = np.arange(256, dtype=np.uint8)
    vals = capi.e4m3_bits_to_f32(allb)
    finite = ~np.isnan(vals)
    assert finite.sum() == 254 and vals[0x7E] == 448.0 and vals[0x01] == 2.0 ** -9 and vals[0x08] == 2.0 ** -6
    # every representable value encodes to itself (−0 keeps its sign bit)
    assert np.array_equal(capi.f32_to_e4m3_bits(vals[finite]), allb[finite])
    # ties to even, saturation, subnormal rounding
    x = np.float32([1.0625, 1.1875, 500.0, -1000.0, 2.0 ** -10, 3 * 2.0 ** -10, 0.0])
    got = capi.e4m3_bits_to_f32(capi.f32_to_e4m3_bits(x))
    assert got.tolist() == [1.0, 1.25, 448.0, -448.0, 0.0, 2 * 2.0 ** -9, 0.0]
    rng = np.random.default_rng(0)
    a = rng.standard_normal((64, 128)).astype(np.float32)
    b, sc = capi.quantize_e4m3(a)
    back = capi.e4m3_bits_to_f32(b) * sc[:, None]
    assert np.abs(back - a).max() <= np.abs(a).max() * 2.0 ** -4   # 3 mantissa bits: half a step of the top binade
