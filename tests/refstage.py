"""Stage an unmodified copy of the reference package with exactly the
`b200` backend INTEGRATION.md section 2 documents (one new file, two
changes in hcub/distributed.py).  Source: baseline/_ref/hcub (the offline
install, travels to the GPU box) or, in the build container,
/root/reference/pkg/src/hcub."""
import os
import re
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref", "hcub"), "/root/reference/pkg/src/hcub")


def reference_source():
    for c in CANDIDATES:
        if os.path.isfile(os.path.join(c, "distributed.py")):
            return c
    return None


def _block(text, marker):
    return text.split(marker, 1)[1].split("```", 1)[0]


def stage(dst):
    """Copy the reference into dst/hcub and apply the documented stub."""
    src = reference_source()
    if src is None:
        raise FileNotFoundError("no reference package (baseline/_ref/hcub)")
    pkg = os.path.join(dst, "hcub")
    shutil.copytree(src, pkg, ignore=shutil.ignore_patterns("__pycache__"))
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    with open(os.path.join(pkg, "b200.py"), "w") as fh:
        fh.write("# hcub/b200.py" + _block(text, "# hcub/b200.py  (new file in the reference package)"))
    lines = _block(text, "# hcub/distributed.py  (two changes)").strip("\n").splitlines()
    backends, body = lines[0].split("  #")[0], [ln for ln in lines[1:] if not ln.strip().startswith("#")]
    p = os.path.join(pkg, "distributed.py")
    code = open(p).read()
    code, n1 = re.subn(r"^BACKENDS = \(.*\)$", backends, code, count=1, flags=re.M)
    anchor = '    raise ValueError(f"unknown backend {backend!r}; expected one of {BACKENDS}")'
    n2 = code.count(anchor)
    code = code.replace(anchor, "\n".join(body) + "\n" + anchor)
    assert n1 == 1 and n2 == 1, "the reference no longer has the documented hook lines"
    open(p, "w").write(code)
    return pkg
