"""CPU tests of the dynamic-topology C ABI (include/cwc_dyn.h): every declared
symbol is exported, model validation errors, the structural classification
and the plan (no compute: there is no GPU here, and the simulate call must
fail loudly without one)."""
import copy
import os
import re

import pytest

import workloads.dynamic as wd
from paper_1010_2438_b200 import cwc, cwc_dyn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1010_2438_b200 import _build
    _build.build()


def test_every_declared_symbol_is_exported():
    hdr = open(os.path.join(ROOT, "include", "cwc_dyn.h")).read()
    declared = set(re.findall(r"\b(cwc_[a-z0-9_]+)\s*\(", hdr))
    L = cwc_dyn.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(cwc_dyn.EXPORTED) == declared


def test_cell_population_compiles():
    m = cwc_dyn.cwc_dyn_model_create(wd.cell_population_model())
    i = cwc_dyn.cwc_dyn_info_get(m)
    assert (i.n_atoms, i.n_labels, i.n_rules, i.n_obs) == (5, 3, 21, 8)
    # structural rules: division, lysis, vesicle formation, fusion, free-vesicle decay, the two no-X rules
    assert i.n_structural == 7
    i = cwc_dyn.cwc_dyn_info_get(m, 8192, 20.0, 0.1)
    assert i.n_stat_cells == 201 * 8 and i.capacity == 64 and i.threads == 128
    assert i.workspace_bytes == cwc_dyn.cwc_dyn_workspace_size(m, 8192, 20.0, 0.1)


@pytest.mark.parametrize("seed", range(40))
def test_random_models_compile(seed):
    cwc_dyn.cwc_dyn_model_create(wd.random_dynamic_model(seed))


def _status(model):
    st, _ = cwc_dyn.cwc_dyn_model_create_status(model)
    return st


def test_validation_errors():
    base = wd.cell_population_model()
    assert _status(base) == cwc.CWC_OK

    m = copy.deepcopy(base)
    m["rules"][0]["rate"] = 0.0
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["rules"][0]["rate"] = float("nan")
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["rules"][1]["atoms"] = {0: 3}            # order 3
    assert _status(m) == cwc.CWC_ERR_UNSUPPORTED
    m = copy.deepcopy(base)
    m["rules"][1]["atoms"] = {9: 1}            # atom out of range
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["rules"][0]["rhs"]["release_Y"] = True   # release without a child pattern
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["rules"][7]["rhs"]["comps"] = [{"label": 1, "wrap": {}, "content": {}, "W": True, "Y": False}]
    assert _status(m) == cwc.CWC_ERR_INVALID   # lysis releases W and a constructor carries it too
    m = copy.deepcopy(base)
    m["rules"][3]["label"] = 7                 # label out of range
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["term"]["comps"][0]["content"]["atoms"] = {0: -1}
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["observables"].append(("wrap", 0, 1))    # wrap of the top level
    assert _status(m) == cwc.CWC_ERR_INVALID
    m = copy.deepcopy(base)
    m["rules"] = m["rules"] * 2                # 42 rules
    assert _status(m) == cwc.CWC_ERR_UNSUPPORTED
    m = copy.deepcopy(base)
    m["term"]["comps"] = [{"label": 1, "wrap": {}, "content": {}}] * 64   # 65 compartments
    assert _status(m) == cwc.CWC_ERR_UNSUPPORTED


def test_run_argument_errors():
    m = cwc_dyn.cwc_dyn_model_create(wd.cell_population_model())
    for args in [(0, 1.0, 0.1), (4, 0.0, 0.1), (4, 1.0, 0.0), (4, 1.0, 2.0)]:
        with pytest.raises(cwc.CwcError) as e:
            cwc_dyn.cwc_dyn_workspace_size(m, *args)
        assert e.value.status == cwc.CWC_ERR_INVALID
    o = cwc_dyn.cwc_dyn_opts()
    o.capacity = 10                            # fewer than the 17 initial compartments
    with pytest.raises(cwc.CwcError):
        cwc_dyn.cwc_dyn_workspace_size(m, 4, 1.0, 0.1, o)
    o = cwc_dyn.cwc_dyn_opts()
    o.replica_offset, o.replicas_total = 10, 12
    with pytest.raises(cwc.CwcError):
        cwc_dyn.cwc_dyn_workspace_size(m, 4, 1.0, 0.1, o)


def test_simulate_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    m = cwc_dyn.cwc_dyn_model_create(wd.cell_population_model())
    with pytest.raises(RuntimeError):
        cwc_dyn.simulate(m, 4, 1.0, 0.1, 1)
    ws = torch.empty(cwc_dyn.cwc_dyn_workspace_size(m, 4, 1.0, 0.1), dtype=torch.uint8)
    st = (torch.empty(88, dtype=torch.int64), torch.empty(88, dtype=torch.int64), torch.empty(176, dtype=torch.int64))
    with pytest.raises(cwc.CwcError) as e:
        cwc_dyn.cwc_dyn_simulate(m, 4, 1.0, 0.1, 1, 0, st, ws)
    assert e.value.status == cwc.CWC_ERR_CUDA
