"""Diagnostic (not part of the test suite): run the reference package's own
test files unmodified against this package, with `lrqbench` aliased to
`paper_2604_26423_b200` (module by module).

    python scripts/run_reference_tests.py <dir with the reference's tests> [pytest args]

The reference's tests are not in this repository; point the script at a copy
(e.g. the one under the git-ignored baseline/_ref/).  Failures are drop-in
gaps or the deviations INTEGRATION.md lists.  `lrqbench.stats` (classify /
fitnoise, out of the hot path's scope) is not implemented here: its names
come from the reference install in baseline/_ref when it is present, so that
test files importing them still collect.
"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODULES = ["circuit", "cli", "engine", "errors", "noise", "problem", "rng", "sharded"]


def main():
    tests = os.path.abspath(sys.argv[1])
    alias = tempfile.mkdtemp(prefix="lrqbench_alias_")
    pkg = os.path.join(alias, "lrqbench")
    os.makedirs(pkg)
    with open(os.path.join(pkg, "__init__.py"), "w") as fh:
        fh.write("import sys\nimport importlib\nimport paper_2604_26423_b200 as _p\n"
                 f"for _m in {MODULES!r}:\n"
                 "    sys.modules['lrqbench.' + _m] = importlib.import_module('paper_2604_26423_b200.' + _m)\n"
                 "sys.modules['lrqbench'] = _p\n"
                 "try:\n"
                 f"    sys.path.append({os.path.join(ROOT, 'baseline', '_ref')!r})\n"
                 "    import importlib.util as _u\n"
                 f"    _spec = _u.spec_from_file_location('lrqbench.stats', {os.path.join(ROOT, 'baseline', '_ref', 'lrqbench', 'stats.py')!r})\n"
                 "    _st = _u.module_from_spec(_spec)\n"
                 "    sys.modules['lrqbench.stats'] = _st\n"
                 "    _spec.loader.exec_module(_st)\n"
                 "    _p.stats = _st\n"
                 "    for _n in getattr(_st, '__all__', [n for n in dir(_st) if not n.startswith('_')]):\n"
                 "        if not hasattr(_p, _n):\n"
                 "            setattr(_p, _n, getattr(_st, _n))\n"
                 "except Exception:\n"
                 "    pass\n")
    env_path = os.pathsep.join([alias, ROOT, os.environ.get("PYTHONPATH", "")])
    os.environ["PYTHONPATH"] = env_path
    args = [sys.executable, "-m", "pytest", tests, "-q", "-p", "no:cacheprovider", "-o", "addopts=",
            "--rootdir", tests, *sys.argv[2:]]
    os.execvpe(args[0], args, os.environ)


if __name__ == "__main__":
    main()
