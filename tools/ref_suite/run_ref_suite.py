#!/usr/bin/env python3
"""Run the reference's own test suite (pkg/tests, 125 tests) against this package.

The reference package `gooms` is imported by its tests as `gooms.core`, `gooms.scan`,
`gooms.lyapunov`, `gooms.ssm`, `gooms.util`, `gooms.systems`, `gooms.oracle`. This
runner installs a `gooms` package in sys.modules whose modules are:

  mode "boundary" (the drop-in as SURVEY §8b draws it): gooms.core and gooms.scan are
      this package's (GPU kernels behind the reference's names); lyapunov, ssm, util,
      systems and oracle are the UNMODIFIED reference modules from the offline install
      (baseline/_ref/gooms), so the reference's own callers run on top of the drop-in;
  mode "full": core, scan, lyapunov and ssm are all this package's.

Names a test imports that this package does not define are filled from the reference
module of the same name and listed in the report (they are host-side helpers outside
the hot path, e.g. the ODE integrator). The reference's test files are staged (not
committed) into baseline/_ref_tests/ by tools/ref_suite/stage.sh in the build container;
both baseline/ directories travel to the GPU box with the snapshot.

  python tools/ref_suite/run_ref_suite.py [--mode boundary|full] [--out report.json]
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref", "gooms")
TESTS = os.path.join(ROOT, "baseline", "_ref_tests")


def _load_ref(name):
    spec = importlib.util.spec_from_file_location(f"gooms.{name}", os.path.join(REF, f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[f"gooms.{name}"] = mod
    spec.loader.exec_module(mod)
    return mod


def install_shim(mode: str):
    sys.path.insert(0, ROOT)
    import paper_2510_03426_b200 as P
    from paper_2510_03426_b200 import core, lyapunov, scan, ssm

    pkg = types.ModuleType("gooms")
    pkg.__path__ = []  # a package: submodules come from sys.modules
    pkg.__package__ = "gooms"
    sys.modules["gooms"] = pkg
    filled = {}

    def alias(name, ours):
        mod = types.ModuleType(f"gooms.{name}")
        mod.__dict__.update({k: v for k, v in vars(ours).items() if not k.startswith("__")})
        mod.__package__ = "gooms"
        sys.modules[f"gooms.{name}"] = mod
        setattr(pkg, name, mod)
        return mod

    util = _load_ref("util")
    pkg.util = util
    ours = {"core": core, "scan": scan}
    if mode == "full":
        ours.update(lyapunov=lyapunov, ssm=ssm)
    for name in ("core", "scan"):
        alias(name, ours[name])
    for name in ("systems", "oracle"):
        setattr(pkg, name, _load_ref(name))
    for name in ("lyapunov", "ssm"):
        if name in ours:
            alias(name, ours[name])
        else:
            setattr(pkg, name, _load_ref(name))
    # fill names the reference modules define and ours do not (reported)
    for name in ("core", "scan", "lyapunov", "ssm"):
        if name not in ours:
            continue
        # the reference module itself (registered under a private name so its relative
        # imports resolve inside the shim package), only to list the names it defines
        spec = importlib.util.spec_from_file_location(f"gooms._ref_{name}",
                                                      os.path.join(REF, f"{name}.py"))
        refmod = importlib.util.module_from_spec(spec)
        sys.modules[f"gooms._ref_{name}"] = refmod
        try:
            spec.loader.exec_module(refmod)
        except Exception as e:  # pragma: no cover
            filled[name] = f"could not load reference module: {e}"
            continue
        mod = sys.modules[f"gooms.{name}"]
        miss = [k for k in vars(refmod) if not k.startswith("__") and k not in vars(mod)
                and not isinstance(getattr(refmod, k), types.ModuleType)]
        for k in miss:
            setattr(mod, k, getattr(refmod, k))
        if miss:
            filled[name] = sorted(miss)
    P._lib.load()
    return filled


class Collect:
    def __init__(self):
        self.results = {}

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            r = {"outcome": report.outcome}
            if report.outcome == "failed":
                r["msg"] = str(report.longrepr)[-1500:]
            self.results[report.nodeid] = r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="boundary", choices=["boundary", "full"])
    ap.add_argument("--out", default=None)
    ap.add_argument("-k", default=None)
    args = ap.parse_args()
    if not os.path.isdir(TESTS) or not os.path.isdir(REF):
        print(json.dumps({"error": "baseline/_ref or baseline/_ref_tests missing "
                                   "(run tools/ref_suite/stage.sh in the build container)"}))
        return 2
    filled = install_shim(args.mode)
    import pytest

    col = Collect()
    pargs = [TESTS, "-q", "-p", "no:cacheprovider", "--rootdir", TESTS]
    if args.k:
        pargs += ["-k", args.k]
    rc = pytest.main(pargs, plugins=[col])
    outcomes = {}
    for r in col.results.values():
        outcomes[r["outcome"]] = outcomes.get(r["outcome"], 0) + 1
    rep = {"mode": args.mode, "rc": int(rc), "counts": outcomes, "filled_from_reference": filled,
           "tests": col.results}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rep, f, indent=1)
    print(json.dumps({"mode": args.mode, "rc": int(rc), "counts": outcomes,
                      "filled_from_reference": filled}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
