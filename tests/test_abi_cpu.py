# SPDX-License-Identifier: Apache-2.0
"""CPU-side checks of the product library: it loads without a GPU, exports
every symbol include/asteria_b200.h declares, and its host-only entry points
(configuration, blocking) match the reference (precond.cpp, config.cpp)."""
import os
import re

import pytest

from paper_2605_16184_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rt():
    from paper_2605_16184_b200 import runtime
    return runtime


def header_symbols():
    text = open(os.path.join(ROOT, "include", "asteria_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(asg_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol(rt):
    syms = header_symbols()
    assert len(syms) >= 39
    for s in syms:
        assert hasattr(rt.lib, s), s
    assert set(syms) == set(rt.EXPORTED)


def test_api_version(rt):
    assert rt.lib.asg_api_version() == 1


def test_no_gpu_means_unsupported(rt):
    # On this CPU-only container the device check says no; creation would
    # fail loudly (there is no CPU fallback).
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert rt.device_supported(0) is False
    with pytest.raises(abi.Error):
        opt = rt.optimizer_defaults(abi.SOAP)
        s = rt.scheduler_defaults()
        s.pf = opt.precondition_frequency
        pd = abi.ParamDesc(0, 0, 4, 4, 4, 4)
        import ctypes as C
        h = C.c_void_p()
        rt.check(rt.lib.asg_blockset_create(0, C.byref(opt), C.byref(s), C.byref(pd), 1, 0, 0, 1, 1, C.byref(h)))


def test_defaults_and_validate(rt):  # precond.cpp:34-62
    a = rt.optimizer_defaults(abi.ADAMW)
    assert a.beta2 == 0.999 and a.accumulation == abi.SUM
    s = rt.optimizer_defaults(abi.SHAMPOO)
    assert s.beta2 == 0.95 and s.accumulation == abi.SUM
    p = rt.optimizer_defaults(abi.SOAP)
    assert p.beta2 == 0.95 and p.accumulation == abi.EMA
    k = rt.optimizer_defaults(abi.KL_SHAMPOO)
    assert k.accumulation == abi.EMA
    for c in (a, s, p, k):
        assert (c.lr, c.beta1, c.eps, c.weight_decay, c.precondition_frequency, c.damping,
                c.block_dim_limit) == (1e-3, 0.9, 1e-8, 0.0, 10, 1e-8, 2048)
        rt.validate(c)
    bad = p.copy()
    bad.beta1 = 1.0
    with pytest.raises(abi.ConfigInvalidError):
        rt.validate(bad)


def test_partition_param_tiles_exactly(rt):  # precond_test.cpp:28-49
    two = rt.partition_param(3000, 500, 2048)
    assert len(two) == 2
    assert (two[0].row_begin, two[0].row_end, two[1].row_begin, two[1].row_end) == (0, 2048, 2048, 3000)
    assert (two[0].col_begin, two[0].col_end) == (0, 500)
    assert len(rt.partition_param(8, 8, 2048)) == 1
    nine = rt.partition_param(5000, 5000, 2048)
    assert len(nine) == 9
    sides = [2048, 2048, 904]
    for r in range(3):
        for c in range(3):
            b = nine[r * 3 + c]
            assert b.rows() == sides[r] and b.cols() == sides[c]
    assert two[1].id("w") == "w[2048:3000,0:500]"


def test_partition_covers_every_index_once(rt):  # precond_test.cpp:51-70
    import numpy as np
    rng = np.random.default_rng(3)
    for _ in range(30):
        rows, cols, limit = int(rng.integers(1, 91)), int(rng.integers(1, 91)), int(rng.integers(1, 41))
        cover = np.zeros((rows, cols))
        for b in rt.partition_param(rows, cols, limit):
            assert b.rows() <= limit and b.cols() <= limit
            cover[b.row_begin:b.row_end, b.col_begin:b.col_end] += 1
        assert cover.min() == 1 and cover.max() == 1
    with pytest.raises(abi.ShapeMismatchError):
        rt.partition_param(0, 3, 2)
    with pytest.raises(abi.ConfigInvalidError):
        rt.partition_param(3, 3, 0)


def test_config_json_reference_files(rt):  # proj/configs/*.json schema, config.cpp:121-205
    qs = open(os.path.join(ROOT, "tests", "golden", "quadratic_shampoo.json")).read()
    o, s, prec = rt.config_from_json(qs)
    assert o.method == abi.SHAMPOO and o.lr == 0.003 and o.accumulation == abi.EMA
    assert o.precondition_frequency == 1 and s.pf == 1 and s.staleness_S == 0
    assert prec == abi.PREC_3XTF32
    cs = open(os.path.join(ROOT, "tests", "golden", "classifier_soap.json")).read()
    o, s, _ = rt.config_from_json(cs)
    assert o.method == abi.SOAP and o.lr == 0.01 and s.staleness_S == 5 and s.inject_job_delay_steps == 3.0
    assert s.drain_budget == 4 and s.step_compute_us == 1000.0 and s.install_cost_us == 10.0


def test_config_json_rules(rt):
    # method defaults apply before overrides (config.cpp:126-127)
    o, s, _ = rt.config_from_json('{"optimizer": {"beta2": 0.5, "method": "SOAP"}}')
    assert o.beta2 == 0.5 and o.accumulation == abi.EMA
    # async.pf defaults to precondition_frequency (config.cpp:140) and must match (config.cpp:42-43)
    o, s, _ = rt.config_from_json('{"optimizer": {"method": "KL-Shampoo", "precondition_frequency": 7}}')
    assert o.method == abi.KL_SHAMPOO and s.pf == 7
    with pytest.raises(abi.ConfigInvalidError):
        rt.config_from_json('{"optimizer": {"precondition_frequency": 7}, "async": {"pf": 3}}')
    with pytest.raises(abi.ConfigInvalidError):
        rt.config_from_json('{"optimizer": {"method": "Adagrad"}}')
    with pytest.raises(abi.ConfigInvalidError):
        rt.config_from_json('{"optimizer": {"accumulation": "Max"}}')
    with pytest.raises(abi.ConfigInvalidError):
        rt.config_from_json('{"optimizer": ')
    # unknown keys/sections are ignored (read_if, config.cpp:12-15); gpu section is additive
    o, s, prec = rt.config_from_json('{"task": {"kind": "x"}, "gpu": {"precision": "tf32", "install_mode": "event"}}')
    assert prec == abi.PREC_TF32 and s.install_mode == abi.INSTALL_EVENT


def test_config_json_gpu_section(rt):
    """The additive "gpu" section: precision, install mode, refresh mode."""
    from paper_2605_16184_b200 import abi
    doc = '{"optimizer": {"method": "SOAP", "precondition_frequency": 4}, "async": {"staleness_S": 2}, ' \
          '"gpu": {"precision": "tf32", "install_mode": "event", "refresh": "f32"}}'
    o, s, p = rt.config_from_json(doc)
    assert o.method == abi.SOAP and o.precondition_frequency == 4 and s.pf == 4 and s.staleness_S == 2
    assert p == abi.PREC_TF32 and s.install_mode == abi.INSTALL_EVENT and s.refresh_mode == abi.REFRESH_F32
    o, s, p = rt.config_from_json('{"optimizer": {"method": "Shampoo"}}')
    assert p == abi.PREC_3XTF32 and s.refresh_mode == abi.REFRESH_F64  # defaults: reference-tight
    with pytest.raises(abi.ConfigInvalidError):
        rt.config_from_json('{"optimizer": {"method": "SOAP"}, "gpu": {"refresh": "f16"}}')
