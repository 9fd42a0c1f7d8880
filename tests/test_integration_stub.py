"""The reference-side binding documented in INTEGRATION.md
(integration/phasemask_gpu.py) agrees with the C ABI: its ctypes structures
have exactly the fields, offsets and sizes of include/phasemask_b200.h's
pm_params / pm_result (parsed from the header) and of the host layer's own
(paper_1302_0120_b200/_lib.py), and INTEGRATION.md shows that file verbatim.
CPU only: the library is loaded, no compute call is made."""

import ctypes as C
import importlib.util
import re
from pathlib import Path

import pytest

from paper_1302_0120_b200 import _lib

REPO = Path(__file__).resolve().parents[1]
CTYPES = {"int": C.c_int, "double": C.c_double, "unsigned long long": C.c_ulonglong}


def header_struct(name):
    """ctypes Structure built from `typedef struct name { ... } name;` of the header."""
    text = (REPO / "include" / "phasemask_b200.h").read_text()
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = " ".join(decl.split())
        if not decl:
            continue
        m = re.fullmatch(r"(const )?(unsigned long long|int|double|float|void|uint8_t)\s+(.*)", decl)
        assert m, decl
        base = m.group(2)
        for d in m.group(3).split(","):                 # `double t_lit, t_dark`
            dm = re.fullmatch(r"\s*(\*?)\s*(\w+)(\[(\d+)\])?\s*", d)
            assert dm, d
            t = C.c_void_p if dm.group(1) else CTYPES[base]
            if dm.group(4):
                t = t * int(dm.group(4))
            fields.append((dm.group(2), t))
    return type(name + "_h", (C.Structure,), {"_fields_": fields})


def layout(st):
    return [(f[0], getattr(st, f[0]).offset, getattr(st, f[0]).size) for f in st._fields_] + [("sizeof", C.sizeof(st))]


def stub_module():
    spec = importlib.util.spec_from_file_location("phasemask_gpu_stub", REPO / "integration" / "phasemask_gpu.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name", ["pm_params", "pm_result"])
def test_stub_structs_match_header_and_host_layer(name):
    h = header_struct(name)
    stub = getattr(stub_module(), name)
    host = getattr(_lib, name)
    assert layout(stub) == layout(h)
    assert layout(host) == layout(h)


def test_integration_md_shows_the_stub_verbatim():
    md = (REPO / "INTEGRATION.md").read_text()
    block = re.search(r"<!-- stub:begin -->\n```python\n(.*?)```\n<!-- stub:end -->", md, re.S).group(1)
    assert block == (REPO / "integration" / "phasemask_gpu.py").read_text()


def test_stub_binds_against_the_built_library():
    lib = stub_module().load(str(_lib.LIB_PATH))
    for sym in ("pm_plan_create", "pm_solve", "pm_last_error"):
        assert hasattr(lib, sym)
