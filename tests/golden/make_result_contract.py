"""Derive tests/golden/result_contract.json from the reference's JSON schema.

The reference validates its run report against proj/docs/result.schema.json (draft-07;
proj/tests/cli_e2e.sh). /root/reference is absent on the GPU box, so this script
flattens the schema into one rule per top-level key -- [key, allowed JSON types,
constraint, element rule] -- which tests/_schema.py checks documents against. It also
stores one report written by the reference itself (oracle/_ref, diam_result_write_json)
so the CPU suite can pin the checker on a document the reference produced.

    python tests/golden/make_result_contract.py
"""
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
SCHEMA = "/root/reference/proj/docs/result.schema.json"


def flatten(node):
    """(types, constraint, element rule) of one schema node."""
    types = node.get("type")
    types = [types] if isinstance(types, str) else list(types or [])
    cons = {}
    if "const" in node:
        cons["equals"] = node["const"]
    if "enum" in node:
        cons["one_of"] = list(node["enum"])
    if "minimum" in node:
        cons["at_least"] = node["minimum"]
    elem = flatten(node["items"]) if "items" in node else None
    return [types, cons, elem]


def main():
    schema = json.load(open(SCHEMA))
    rules = [[key] + flatten(node) for key, node in schema["properties"].items()]
    out = {"source": "derived from proj/docs/result.schema.json by make_result_contract.py",
           "document_type": schema["type"], "mandatory": sorted(schema["required"]),
           "closed": schema.get("additionalProperties") is False, "rules": rules}
    with open(os.path.join(HERE, "result_contract.json"), "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")

    import _oracle as O  # noqa: E402
    from paper_1506_05741_b200.abi import DiamABI  # noqa: E402
    ref = DiamABI(O.REF_SO)
    t = ref.target_build("pi2", 6, 2)
    r = ref.sample(t, kernel="diam", chains=2, intervals_per_batch=2, max_batches=3, n_lag=10, n0=5, master_seed=3,
                   threads=1)
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "r.json")
        r.write_json(p)
        doc = json.load(open(p))
    with open(os.path.join(HERE, "ref_result.json"), "w") as f:
        json.dump(doc, f)
        f.write("\n")


if __name__ == "__main__":
    main()
