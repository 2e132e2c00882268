"""The C-ABI library without a GPU: it loads, exports every symbol
include/pclab_b200.h declares, and its host-only entry points (status names,
models, checkpoints, seeded fields) behave like the reference's
(capi.cpp, gnn.cpp:226-249, rng.hpp). No compute call needs CUDA here."""
import json
import os

import numpy as np
import pytest

import paper_2412_07127_b200 as P
from conftest import bits
from oracle import oracle as O


def test_library_loads_and_exports_header():
    L = P.lib()
    syms = P.exported_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert missing == []
    # the reference's C entry points (pclab.h) are all present under their names
    for s in ("pclab_version", "pclab_status_name", "pclab_last_error", "pclab_matrix_read",
              "pclab_matrix_write", "pclab_matrix_from_coo", "pclab_matrix_gen_poisson",
              "pclab_matrix_shape", "pclab_matrix_free", "pclab_model_init", "pclab_model_load",
              "pclab_model_save", "pclab_model_param_count", "pclab_model_free", "pclab_pcg_solve",
              "pclab_run", "pclab_string_free"):
        assert s in syms


def test_status_names_match_reference():
    names = [P.lib().pclab_status_name(i).decode() for i in range(6)]
    assert names == ["ok", "argument", "format", "numeric", "io", "internal"]
    assert P.lib().pclab_last_error() is not None


def test_model_init_matches_reference_and_roundtrips(tmp_path):
    m = P.Model.init(1)
    assert m.param_count() == 997
    assert np.array_equal(bits(m.params()), bits(O.gnn_init(1)))
    path = str(tmp_path / "ck.json")
    m.save(path)
    j = json.load(open(path))
    assert j["format"] == "pclab-gnn" and j["version"] == 1 and len(j["params"]) == 997
    m2 = P.Model.load(path)
    assert np.array_equal(bits(m2.params()), bits(m.params()))


def test_model_load_errors(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"format": "other", "version": 1, "params": []}))
    with pytest.raises(P.FormatError, match="format tag"):
        P.Model.load(str(bad))
    bad.write_text(json.dumps({"format": "pclab-gnn", "version": 1, "hidden": 8, "blocks": 3,
                               "node_features": 9, "params": [0.0] * 10}))
    with pytest.raises(P.FormatError, match="parameter count"):
        P.Model.load(str(bad))
    with pytest.raises(P.IoError):
        P.Model.load(str(tmp_path / "missing.json"))
    with pytest.raises(P.ArgumentError):
        P.Model.from_params(np.zeros(10))


def test_reference_checkpoint_format_loads(tmp_path):
    """A checkpoint in the reference's exact layout (model_to_json dump(2))."""
    p = O.gnn_init(7)
    path = tmp_path / "ref.json"
    path.write_text(json.dumps({"blocks": 3, "format": "pclab-gnn", "hidden": 8, "node_features": 9,
                                "params": p.tolist(), "version": 1}, indent=2))
    assert np.array_equal(bits(P.Model.load(str(path)).params()), bits(p))


def test_seeded_fields_match_oracle():
    assert P.uniform_at(5, 9) == O.uniform_at(5, 9)
    assert P.derive_seed(3, 14) == O.derive_seed(3, 14)
    assert np.array_equal(bits(P.field_normal(1000, 4)), bits(O.normal_field(1000, 4)))
    assert np.array_equal(bits(P.field_lognormal(1000, 4, 1.5)), bits(O.lognormal_field(1000, 4, 1.5)))
    assert np.array_equal(bits(P.field_uniform_pm1(1000, 4)), bits(O.uniform_pm1_field(1000, 4)))


def test_run_is_outside_the_path():
    with pytest.raises(P.ArgumentError, match="outside the accelerated"):
        P.run("train", {})


def test_workload_inputs_match_oracle():
    for w in P.workloads.CONFIGS:
        s = w.scaled(3)
        if s.family == "elasticity":
            assert np.array_equal(bits(P.workloads.moduli(s, P.field_lognormal, P.derive_seed)),
                                  bits(P.workloads.moduli(s, O.lognormal_field, O.derive_seed)))
    assert P.workloads.CONFIGS[2].n == 5012994 and P.workloads.CONFIGS[3].n == 10057500
