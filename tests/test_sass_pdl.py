"""Static check of the built library (CPU; needs cuobjdump): in every kernel that waits on its
programmatic-dependent-launch predecessor (griddepcontrol.wait = SASS ACQBULK), no global load
(LDG) may be scheduled before that wait -- a load hoisted above it can read data the predecessor
has not written yet (found in round 2: a `const __restrict__` length read compiled to
LDG.E.CONSTANT above ACQBULK).  Intentional early reads go through cp.async / TMA (LDGSTS,
UTMALDG: weights, which no kernel writes) and are not flagged; decode_step_kernel and
m2_scan_kernel are exempt by name: their pre-wait LDGs are the layer's a_log / b_dt (dt_bias) / D
entries, read before griddepcontrol.wait on purpose ("weights first"), never written by a kernel."""
import os
import shutil
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_21144_b200", "libssmtp.so")


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not os.path.exists(LIB), reason="cuobjdump / library missing")
def test_no_global_load_before_pdl_wait():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    bad, fn, waited, has_wait, early = [], None, False, False, []
    funcs = []
    for line in out.splitlines():
        if "Function :" in line:
            if fn is not None:
                funcs.append((fn, has_wait, early))
            fn, waited, has_wait, early = line.split("Function :")[1].strip(), False, False, []
            continue
        if "ACQBULK" in line:
            waited = has_wait = True
        tok = line.split(";")[0].split()
        ops = [t for t in tok if t.startswith("LDG") and not t.startswith(("LDGSTS", "LDGDEPBAR"))]
        if ops and not waited:
            early.append(ops[0])
    if fn is not None:
        funcs.append((fn, has_wait, early))
    exempt = ("decode_step_kernel", "m2_scan_kernel")
    bad = [(f, e) for f, w, e in funcs if w and e and not any(x in f for x in exempt)]
    assert funcs, "no kernels found"
    assert not bad, bad
