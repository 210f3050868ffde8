"""The product path never touches the oracle, and fails loudly without its
native build (CPU, static checks on the package sources)."""

import ast
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2602_21548_b200")


def test_package_python_never_imports_the_oracle():
    for name in os.listdir(PKG):
        if not name.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(PKG, name)).read())
        for node in ast.walk(tree):
            mods = []
            if isinstance(node, ast.Import):
                mods = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                mods = [node.module or ""]
            assert not any(m.split(".")[0] == "oracle" for m in mods), f"{name} imports the oracle"


def test_native_sources_never_link_the_oracle():
    pat = re.compile(r'#include\s*"[^"]*(kvref|ref_shim|oracle)[^"]*"|dlopen|libkvref|libpdsim_ref')
    for sub in ("csrc",):
        for name in os.listdir(os.path.join(PKG, sub)):
            text = open(os.path.join(PKG, sub, name)).read()
            assert not pat.search(text), f"{sub}/{name} references the oracle"
    mk = "\n".join(l for l in open(os.path.join(PKG, "Makefile")).read().splitlines()
                   if not l.lstrip().startswith("#"))
    assert "oracle" not in mk and "kvref" not in mk


def test_package_requires_its_native_build():
    init = open(os.path.join(PKG, "__init__.py")).read()
    # the extension import is unconditional and re-raised with a build hint
    assert "from ._core import" in init and "raise ImportError" in init
    abi = open(os.path.join(PKG, "abi.py")).read()
    assert "raise ImportError" in abi  # libdualpath.so missing -> loud failure
