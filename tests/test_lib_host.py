"""CPU-side checks of the native library: it loads, exports every symbol the
header declares, and its host-only logic (binomial schedule, problem
validation, workspace planning) matches the oracle / reference semantics."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import revolve as orv
from paper_2206_01298_b200 import _lib
from paper_2206_01298_b200 import policies
from paper_2206_01298_b200.configs import make_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import os
    if not os.path.exists(_lib.LIB_PATH):      # CPU container: build once if absent
        from paper_2206_01298_b200 import build
        build.build()
    return _lib.load()


def test_library_exports_every_header_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "odeblock.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(ob_\w+)\(", hdr, re.M))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert "sm_100a" in _lib.version()


def test_revolve_count_matches_oracle(lib):
    for nt in range(1, 61):
        for nc in range(1, 21):
            assert policies.revolve_count(nt, nc) == orv.revolve_count(nt, nc)


def test_revolve_schedule_matches_reference_golden(lib, golden):
    g = golden("revolve.npz")
    kinds = {"advance": 0, "store": 1, "restore": 2, "reverse": 3}
    for key, arr in g.items():
        if not key.startswith("sched_"):
            continue
        _, nt, nc = key.split("_")
        acts = policies.revolve_schedule(int(nt), int(nc))
        mine = np.array([[kinds[a.kind], a.step, a.start, a.stop] for a in acts], np.int64)
        assert np.array_equal(mine, arr), key


def test_revolve_schedule_matches_oracle_grid(lib):
    for nt in range(1, 45):
        for nc in range(1, 12):
            a = [(x.kind, x.step, x.start, x.stop) for x in policies.revolve_schedule(nt, nc)]
            assert a == orv.revolve_schedule(nt, nc), (nt, nc)


def test_invalid_schedule_arguments(lib):
    with pytest.raises(ValueError):
        policies.revolve_count(0, 1)
    with pytest.raises(ValueError):
        policies.revolve_schedule(5, 0)
    with pytest.raises(ValueError):
        policies.CheckpointPolicy("revolve", 0)
    with pytest.raises(ValueError):
        policies.CheckpointPolicy("keep_everything")
    assert policies.CheckpointPolicy.parse("revolve:5").nc == 5


def _problem(ci, policy="store_all"):
    from paper_2206_01298_b200.controls import SolverConfig
    from paper_2206_01298_b200.schemes import tableau_catalog, to_desc

    p = _lib.Problem()
    f = p.field
    f.kind = _lib.OB_FIELD_MLP
    f.dtype = _lib.OB_F32 if ci.dtype == "f32" else _lib.OB_F64
    f.n_layers = len(ci.widths) - 1
    for i, w in enumerate(ci.widths):
        f.widths[i] = w
    f.activation = 2
    f.time_input = int(ci.time_input)
    f.n_params = ci.theta.size
    p.scheme = to_desc(tableau_catalog(ci.scheme))
    p.solver = SolverConfig().to_desc()
    p.batch = p.batch_global = ci.batch
    p.n_steps = ci.n_steps
    pol = policies.CheckpointPolicy.parse(policy)
    p.policy = _lib.OB_POLICY[pol.kind]
    p.nc = pol.nc
    ts = np.linspace(ci.t0, ci.tF, ci.n_steps + 1)
    p.times = ts.ctypes.data_as(C.POINTER(C.c_double))
    return p, ts


@pytest.mark.parametrize("name,pol", [("C1", "store_all"), ("C2", "revolve:8"),
                                      ("C2", "store_all"), ("C2", "store_solutions")])
def test_workspace_planning(lib, name, pol):
    ci = make_config(name)
    p, _ts = _problem(ci, pol)
    n = C.c_size_t()
    assert lib.ob_grad_workspace_size(C.byref(p), C.byref(n)) == _lib.OB_OK
    esz = 4 if ci.dtype == "f32" else 8
    state = ci.batch * ci.widths[-1] * esz
    s = 7 if ci.scheme == "dopri5" else 4
    if pol == "store_all":
        assert n.value >= ci.n_steps * (s + 1) * state
    if pol.startswith("revolve"):
        # nc + 1 record buffers at most (slots + the record in hand) + 1 spare
        assert n.value < (8 + 3) * (s + 1) * state + 512 * 2**20


def test_validation_errors_map_to_value_error(lib):
    ci = make_config("C1", batch=4)
    p, _ts = _problem(ci)
    p.field.widths[0] = 65          # inconsistent with time_input=0
    n = C.c_size_t()
    assert lib.ob_grad_workspace_size(C.byref(p), C.byref(n)) == _lib.OB_ERR_VALUE
    assert "inconsistent" in _lib.last_error()
    p, _ts = _problem(ci)
    p.field.n_params += 1
    assert lib.ob_grad_workspace_size(C.byref(p), C.byref(n)) == _lib.OB_ERR_VALUE
    p, ts = _problem(ci)
    ts[3] = ts[2]                   # zero step
    assert lib.ob_grad_workspace_size(C.byref(p), C.byref(n)) == _lib.OB_ERR_VALUE
