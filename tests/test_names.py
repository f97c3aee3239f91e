"""Static check (CPU): no function refers to a global name that no module
statement defines -- the NameError class of bug that only shows up when a
rarely-taken branch runs on the GPU box (bench.py's round-2 `count_flags`
slip failed four GPU tests).  symtable resolves the scopes; no linter is
installed in this image."""

import builtins
import glob
import os
import symtable

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = sorted(
    [os.path.join(ROOT, f) for f in ("bench.py", "bench_cpu.py", "__graft_entry__.py")]
    + glob.glob(os.path.join(ROOT, "paper_2412_16370_b200", "*.py"))
    + glob.glob(os.path.join(ROOT, "oracle", "*.py"))
    + glob.glob(os.path.join(ROOT, "tests", "*.py")))


def _undefined(path):
    with open(path) as f:
        top = symtable.symtable(f.read(), path, "exec")
    defined = set(dir(builtins)) | {"__file__", "__name__", "__doc__", "__spec__"}
    for sym in top.get_symbols():
        if sym.is_assigned() or sym.is_imported() or sym.is_namespace():
            defined.add(sym.get_name())

    def walk(t, out):
        for ch in t.get_children():
            for sym in ch.get_symbols():
                if sym.is_declared_global() and sym.is_assigned():
                    defined.add(sym.get_name())
            walk(ch, out)

    def check(t, out):
        for ch in t.get_children():
            for sym in ch.get_symbols():
                if sym.is_global() and sym.is_referenced() and sym.get_name() not in defined:
                    out.append(f"{ch.get_name()}: {sym.get_name()}")
            check(ch, out)

    out = []
    walk(top, out)
    check(top, out)
    return out


@pytest.mark.parametrize("path", FILES, ids=[os.path.relpath(p, ROOT) for p in FILES])
def test_no_undefined_globals(path):
    assert _undefined(path) == []
