"""Print numpy's SVML pow constant table (__svml_dpow_ha_data_internal_avx512)
as the C initialisers used in paper_2508_09591_b200/csrc/numpy_pow.cuh.

The table lives in numpy's _multiarray_umath extension (numpy 2.3.x, x86-64,
AVX512_SKX build).  Offsets follow the main path of __svml_pow8_ha.
"""

import glob
import struct
import subprocess
import sys

import numpy as np


def main():
    so = glob.glob(str(__import__("pathlib").Path(np.__file__).parent / "_core" /
                       "_multiarray_umath*.so"))[0]
    syms = subprocess.run(["nm", so], capture_output=True, text=True).stdout
    addr = next(int(l.split()[0], 16) for l in syms.splitlines()
                if l.endswith(" __svml_dpow_ha_data_internal_avx512"))
    hdr = subprocess.run(["objdump", "-h", so], capture_output=True, text=True).stdout
    ro = next(l.split() for l in hdr.splitlines() if " .rodata " in l)
    vma, fileoff = int(ro[3], 16), int(ro[5], 16)
    data = open(so, "rb").read()
    base = addr - vma + fileoff
    vec = {"kLogHiA": 0x000, "kLogHiB": 0x080, "kLogLoA": 0x100, "kLogLoB": 0x180,
           "kExpHi": 0x200, "kExpLo": 0x280}
    for name, off in vec.items():
        v = struct.unpack("<16Q", data[base + off: base + off + 128])
        print(f"{name}: " + ", ".join(f"0x{x:016x}ull" for x in v))
    for off in range(0x300, 0x9c1, 0x40):
        (v,) = struct.unpack("<Q", data[base + off: base + off + 8])
        print(f"0x{off:03x}: 0x{v:016x}ull")


if __name__ == "__main__":
    sys.exit(main())
