"""CPU-side checks of the drop-in boundary: the C-ABI library loads (no GPU
needed) and exports exactly what include/hcub_b200.h declares; host-side
geometry/rule metadata match the reference semantics."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "hcub_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?(?:int|void|char\s*\*|const char\s*\*)\s*\**\s*(hcub_\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("hcub_integrate", "hcub_apply_rule_batch", "hcub_worker_evaluate", "hcub_worker_classify",
                 "hcub_worker_take_top", "hcub_worker_append", "hcub_abi_version"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2511_01573_b200 import _lib
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(_lib.SIGNATURES) == set(declared_functions())
    assert L.hcub_abi_version() == 2


def test_ctypes_struct_layout_matches_header(tmp_path):
    """sizeof/offsetof of every ABI struct, from the C header compiled with
    gcc, equal the ctypes mirrors."""
    import ctypes as C
    import subprocess
    from paper_2511_01573_b200 import _lib
    structs = {"hcub_integrand": _lib.hcub_integrand, "hcub_rule": _lib.hcub_rule,
               "hcub_driver_cfg": _lib.hcub_driver_cfg, "hcub_result": _lib.hcub_result,
               "hcub_classify_out": _lib.hcub_classify_out}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'  printf("{name} %zu\\n", sizeof({name}));')
        for fname, _ in cls._fields_:
            lines.append(f'  printf("{name}.{fname} %zu\\n", offsetof({name}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.splitlines())
    for name, cls in structs.items():
        assert int(got[name]) == C.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert int(got[f"{name}.{fname}"]) == getattr(cls, fname).offset, (name, fname)


def test_gm_rule_metadata_matches_oracle():
    import paper_2511_01573_b200 as hb
    from oracle import hcub_oracle as orc
    for d in range(2, 14):
        t = hb.build_gm_rule(d)
        o = orc.gm_table(d)
        assert t.node_count == o.K
        assert t.fourth_diff_ratio == o.ratio
        assert t.null_center_weight == o.null_center and t.null_axis_weight == o.null_axis
        if d <= 9:
            assert np.array_equal(t.points, o.points)
            assert np.array_equal(t.weights, o.w) and np.array_equal(t.embedded_weights, o.we)


def test_unsupported_dimension():
    import paper_2511_01573_b200 as hb
    with pytest.raises(hb.UnsupportedDimensionError):
        hb.build_gm_rule(14)
    with pytest.raises(hb.UnsupportedDimensionError):
        hb.build_gk_tensor_rule(7)


def test_arbitrary_callables_rejected():
    import paper_2511_01573_b200 as hb
    from paper_2511_01573_b200.integrands import device_descriptor
    with pytest.raises(TypeError):
        device_descriptor(lambda x: x[:, 0], 3)


def test_reference_integrals_match_survey():
    import paper_2511_01573_b200 as hb
    assert hb.reference_integral("f2", 5)[0] == pytest.approx(84065401179.140671, rel=1e-15)
    assert hb.reference_integral("f2", 8)[0] == pytest.approx(3.0156967210413069e17, rel=1e-15)
    assert hb.reference_integral("f4", 3)[0] == pytest.approx(3.5637299179722912e-4, rel=1e-15)
    assert hb.reference_integral("f3", 10)[0] == pytest.approx(2.8026138247446969e-14, rel=1e-15)
    assert hb.reference_integral("f6", 6)[0] == pytest.approx(154773678.85091206, rel=1e-15)


def test_partition_matches_oracle():
    import paper_2511_01573_b200 as hb
    from paper_2511_01573_b200.regions import partition_arrays
    from oracle import hcub_oracle as orc
    for d, k in [(3, 6), (8, 64), (5, 10), (4, 24)]:
        lo, hi = partition_arrays(hb.HyperRect.unit_cube(d), k)
        olo, ohi = orc.partition(np.zeros(d), np.ones(d), k)
        assert np.array_equal(lo, olo) and np.array_equal(hi, ohi)


def test_k1_lane_knob_validates_without_a_gpu():
    """hcub_set_k1_lanes touches no CUDA state: range errors map to ValueError
    (HCUB_E_ARG) like the reference's bad-argument errors."""
    import paper_2511_01573_b200 as hb
    with pytest.raises(ValueError):
        hb.set_k1_lanes(6)
    with pytest.raises(ValueError):
        hb.set_k1_lanes(-2)
    hb.set_k1_lanes(0)
    hb.set_k1_lanes(-1)


def test_integration_stub_structs_match_the_abi():
    """The ctypes stub INTEGRATION.md shows a reference maintainer declares
    structs with the same layout as the library's own bindings."""
    import ctypes as C
    from paper_2511_01573_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = text.split("# hcub/b200_ctypes.py", 1)[1].split("\n", 1)[1].split("```", 1)[0]  # the raw ctypes stub
    keep = []
    for line in code.splitlines():
        if line.startswith(("import", "from", "_lib =", "def ")):
            if line.startswith("def "):
                break
            continue
        keep.append(line)
    ns = {"C": C, "np": np}
    exec("\n".join(keep), ns)
    for stub, mine in (("_Integrand", _lib.hcub_integrand), ("_Rule", _lib.hcub_rule), ("_Cfg", _lib.hcub_driver_cfg),
                       ("_Result", _lib.hcub_result)):
        assert C.sizeof(ns[stub]) == C.sizeof(mine), stub
        assert [f[0] for f in ns[stub]._fields_] == [f[0] for f in mine._fields_], stub
