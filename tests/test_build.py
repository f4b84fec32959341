"""Build-level guards (CPU): the default dense-sweep kernels compile
without register spills (a spill in union_kernel cost 5% on config 2)."""
import os
import re

from conftest import ROOT

LOG = os.path.join(ROOT, "paper_1011_5599_b200", "csrc", "build", "hanf_kernels.o.ptxas.log")

# mangled template arguments of the default dense variants: R, NREG, U, GMODE,
# kVec16, MINB, PF, SKIP=false (hanf_kernels.cu launch_union)
DEFAULTS = ["ILi5ELi64ELi2ELi1ELb0ELi5ELb1ELb0E",   # m = 64 (configs 5; 1, 2 under HANF_LAYOUT=packed)
            "ILi5ELi32ELi4ELi3ELb0ELi1ELb1ELb0E",   # m = 32, padded rows (config 4)
            "ILi5ELi128ELi2ELi0ELb1ELi3ELb1ELb0E"]  # m = 128 (config 3)


def test_default_union_kernels_do_not_spill(hanf):
    text = open(LOG).read()
    for tag in DEFAULTS:
        m = re.search(r"union_kernel" + tag + r"EEvNS_9UnionArgsE' for 'sm_100a'\n[^\n]*\n\s*(\d+) bytes "
                      r"stack frame, (\d+) bytes spill stores", text)
        assert m, tag
        assert int(m.group(2)) == 0, (tag, m.group(0))
