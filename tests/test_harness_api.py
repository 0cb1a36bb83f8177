"""Every scn_harness / binding name the GPU tests, examples, bench and smoke use exists
(CPU check: the GPU suite itself only runs on the B200 box)."""
import glob
import os
import re

import paper_1805_07339_b200 as scn
import scn_harness

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _users():
    files = glob.glob(os.path.join(ROOT, "tests", "**", "*.py"), recursive=True)
    files += glob.glob(os.path.join(ROOT, "examples", "*.py"))
    files += [os.path.join(ROOT, "bench.py"), os.path.join(ROOT, "__graft_entry__.py")]
    return files


def test_harness_names_exist():
    missing = set()
    for f in _users():
        for name in re.findall(r"\bscn_harness\.(\w+)", open(f).read()):
            if name == "py":  # file names
                continue
            if not hasattr(scn_harness, name):
                missing.add((os.path.relpath(f, ROOT), name))
    assert not missing, sorted(missing)


def test_binding_names_exist():
    missing = set()
    for f in _users() + [os.path.join(ROOT, "scn_harness.py")]:
        for name in re.findall(r"\bscn\.(scn_\w+|SCN_\w+)", open(f).read()):
            if not hasattr(scn, name):
                missing.add((os.path.relpath(f, ROOT), name))
    assert not missing, sorted(missing)
