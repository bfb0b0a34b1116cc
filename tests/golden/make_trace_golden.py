"""Generate tests/golden/trace.json from the LIVE reference (build container only).

    python tests/golden/make_trace_golden.py

The reference writes the EDGT trace of TRACE_SPEC (grad_source.write_trace,
grad_source.py:51-74) and runs its own ``analyze-trace`` command on it
(cli.cmd_analyze_trace, cli.py:600-659) with both estimators; the fixture
holds the trace file's sha256 and the three CSVs verbatim.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from edgc import cli as rcli  # noqa: E402  (the reference)
from edgc import grad_source as rgs  # noqa: E402

from tests.golden.specs import TRACE_SPEC, trace_frames  # noqa: E402

CSVS = ("entropy_windows.csv", "gradient_histograms.csv", "layer_correlations.csv")


def main():
    out = {"spec": TRACE_SPEC, "runs": {}}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "t.edgt")
        rgs.write_trace(path, trace_frames())
        with open(path, "rb") as fh:
            out["trace_sha256"] = hashlib.sha256(fh.read()).hexdigest()
        for est in ("histogram", "gaussian"):
            od = os.path.join(tmp, est)
            cfg = {"seed": 3, "output_dir": od, "source": {"trace": path},
                   "sampler": {"alpha": TRACE_SPEC["alpha"], "beta": TRACE_SPEC["beta"]},
                   "window": TRACE_SPEC["window"], "estimator": est,
                   "correlation_iterations": TRACE_SPEC["correlation_iterations"]}
            assert rcli.cmd_analyze_trace(cfg) == 0
            out["runs"][est] = {name: open(os.path.join(od, name)).read() for name in CSVS}
    with open(os.path.join(HERE, "trace.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
