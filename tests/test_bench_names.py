"""bench.py and __graft_entry__.py run only on the GPU box; catch unbound
names (a renamed parameter, a missing import) here on CPU with symtable:
every implicitly-global name a function reads must be a module global or a
builtin."""
import builtins
import symtable
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def unbound(path):
    src = path.read_text()
    top = symtable.symtable(src, str(path), "exec")
    module_names = {s.get_name() for s in top.get_symbols() if s.is_assigned() or s.is_imported()}
    bad = []

    def walk(t):
        for s in t.get_symbols():
            if t.get_type() != "module" and s.is_global() and s.is_referenced():
                n = s.get_name()
                if n not in module_names and not hasattr(builtins, n):
                    bad.append(f"{t.get_name()}:{n}")
        for c in t.get_children():
            walk(c)

    walk(top)
    return bad


@pytest.mark.parametrize("name", ["bench.py", "__graft_entry__.py"])
def test_no_unbound_names(name):
    assert unbound(ROOT / name) == []
