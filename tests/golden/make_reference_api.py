"""Record the reference's renewal-path API surface (field names, order and
defaults of `RenewalConfig`, the `Strategy` members) from /root/reference,
so the GPU box — where the reference does not exist — can build config
objects that carry exactly the reference's fields (tests/test_boundary.py).

    python tests/golden/make_reference_api.py
"""

from __future__ import annotations

import dataclasses
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from spreadsim import renewal as R  # noqa: E402
from spreadsim.graph import Strategy  # noqa: E402


def main() -> None:
    fields = []
    for f in dataclasses.fields(R.RenewalConfig):
        d = f.default
        fields.append({"name": f.name, "default": d.name if isinstance(d, Strategy) else d})
    api = {"RenewalConfig": fields, "Strategy": {m.name: m.value for m in Strategy},
           "source": "spreadsim.renewal.RenewalConfig (R/renewal.py:75-99), spreadsim.graph.Strategy (R/graph.py:61-67)"}
    (OUT / "reference_api.json").write_text(json.dumps(api, indent=1))
    print(json.dumps(api))


if __name__ == "__main__":
    main()
