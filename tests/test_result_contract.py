"""The run report's JSON contract (the report must validate against
proj/docs/result.schema.json). CPU: the checker accepts the reference's own report and
rejects broken ones; the flattened contract equals a fresh derivation from the reference's
schema when /root/reference is present. The GPU engine's reports are checked in
tests/test_gpu_sampler.py::test_json_report_matches_contract."""
import copy
import json
import os

import pytest

import _schema

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_report_satisfies_contract():
    doc = json.load(open(os.path.join(GOLD, "ref_result.json")))
    assert _schema.violations(doc) == []


@pytest.mark.parametrize("mutate,needle", [
    (lambda d: d.pop("ess"), "missing key ess"),
    (lambda d: d.__setitem__("extra", 1), "unexpected key extra"),
    (lambda d: d.__setitem__("kernel", "hmc"), "kernel"),
    (lambda d: d.__setitem__("schema", "diam-run-result/2"), "schema"),
    (lambda d: d.__setitem__("dim", 1), "dim"),
    (lambda d: d.__setitem__("batches", 2.5), "batches"),
    (lambda d: d.__setitem__("stop_reason", "converged"), "stop_reason"),
    (lambda d: d["beta_history"][0].__setitem__(0, None), "beta_history[0][0]"),
    (lambda d: d.__setitem__("global_mean", [1.0, "x"]), "global_mean[1]"),
])
def test_contract_rejects_broken_reports(mutate, needle):
    doc = copy.deepcopy(json.load(open(os.path.join(GOLD, "ref_result.json"))))
    mutate(doc)
    errs = _schema.violations(doc)
    assert errs and any(needle in e for e in errs), errs


@pytest.mark.skipif(not os.path.exists("/root/reference/proj/docs/result.schema.json"),
                    reason="reference tree absent (GPU box)")
def test_contract_is_the_reference_schema():
    import sys
    sys.path.insert(0, GOLD)
    import make_result_contract as m
    schema = json.load(open(m.SCHEMA))
    c = json.load(open(_schema.CONTRACT))
    assert c["mandatory"] == sorted(schema["required"])
    assert c["rules"] == [[k] + m.flatten(v) for k, v in schema["properties"].items()]
    assert c["closed"] == (schema["additionalProperties"] is False)
