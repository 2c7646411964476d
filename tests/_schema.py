"""Checker for the run report's JSON contract (tests/golden/result_contract.json, derived
from the reference's proj/docs/result.schema.json by tests/golden/make_result_contract.py).
Implements the draft-07 subset that schema uses: type (integer / number / string / array /
object / null), const, enum, minimum, array items, required keys, no additional keys."""
import json
import os

CONTRACT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "result_contract.json")


def _is_type(v, t):
    if t == "null":
        return v is None
    if t == "integer":
        return isinstance(v, int) and not isinstance(v, bool)
    if t == "number":
        return isinstance(v, (int, float)) and not isinstance(v, bool)
    if t == "string":
        return isinstance(v, str)
    if t == "array":
        return isinstance(v, list)
    if t == "object":
        return isinstance(v, dict)
    if t == "boolean":
        return isinstance(v, bool)
    raise ValueError(t)


def _check(v, rule, where, errors):
    types, cons, elem = rule
    if types and not any(_is_type(v, t) for t in types):
        errors.append(f"{where}: {type(v).__name__} is not {types}")
        return
    if "equals" in cons and v != cons["equals"]:
        errors.append(f"{where}: {v!r} != {cons['equals']!r}")
    if "one_of" in cons and v not in cons["one_of"]:
        errors.append(f"{where}: {v!r} not in {cons['one_of']}")
    if "at_least" in cons and _is_type(v, "number") and v < cons["at_least"]:
        errors.append(f"{where}: {v} < {cons['at_least']}")
    if elem is not None and isinstance(v, list):
        for i, e in enumerate(v):
            _check(e, elem, f"{where}[{i}]", errors)


def violations(doc, contract=None):
    """List of contract violations of a parsed report (empty = valid)."""
    c = contract or json.load(open(CONTRACT))
    errors = []
    if not _is_type(doc, c["document_type"]):
        return [f"document is not an {c['document_type']}"]
    for key in c["mandatory"]:
        if key not in doc:
            errors.append(f"missing key {key}")
    rules = {r[0]: r[1:] for r in c["rules"]}
    for key, v in doc.items():
        if key not in rules:
            if c["closed"]:
                errors.append(f"unexpected key {key}")
            continue
        _check(v, rules[key], key, errors)
    return errors
