"""Every Python call site of a C-ABI entry point passes exactly the number of
arguments `_native.SIGNATURES` (and so include/mxb200.h) declares.

ctypes accepts surplus arguments silently, so a call written against a
different revision of the ABI would bind its stream argument wrongly; this
static check catches that on CPU, the strict wrapper in `_native.load()`
catches it at run time."""

import ast
import os

from paper_2411_09510_b200._native import SIGNATURES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCAN = ("paper_2411_09510_b200", "scripts", "tests", "bench.py", "__graft_entry__.py")


def _py_files():
    for entry in SCAN:
        path = os.path.join(ROOT, entry)
        if os.path.isfile(path):
            yield path
            continue
        for dirpath, _dirs, files in os.walk(path):
            for f in files:
                if f.endswith(".py"):
                    yield os.path.join(dirpath, f)


def test_call_sites_match_declared_arity():
    bad, seen = [], 0
    for path in _py_files():
        tree = ast.parse(open(path).read(), filename=path)
        for node in ast.walk(tree):
            if not (isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute)):
                continue
            name = node.func.attr
            if name not in SIGNATURES:
                continue
            if any(isinstance(a, ast.Starred) for a in node.args) or node.keywords:
                continue  # arity not static
            seen += 1
            want = len(SIGNATURES[name][1])
            if len(node.args) != want:
                bad.append(f"{os.path.relpath(path, ROOT)}:{node.lineno} {name}: "
                           f"{len(node.args)} args, ABI declares {want}")
    assert seen > 20
    assert not bad, "\n".join(bad)
