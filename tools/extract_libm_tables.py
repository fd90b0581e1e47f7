"""Provenance of the constants in paper_2605_08699_b200/csrc/libm_restated.cuh.

Reads them out of the binaries the reference's arithmetic runs on in this
image and checks them against the header:
  * numpy 2.3 _multiarray_umath: Intel SVML __svml_exp8_ha / __svml_log8_ha
    data blocks (__svml_dexp_ha_data_internal_avx512,
    __svml_dlog_ha_data_internal_avx512; located through the exp8 shift
    constant 0x1.8000000003ff0p+48 and the log threshold 0.75 table);
  * glibc libm: __exp_data.tab (2^(k/128) as tail / head - (k << 45)).
The vrcp14pd step thresholds are probed by tools/rcp14_probe.c
(gcc -O2 -mavx512f; needs an AVX-512 host).

    python tools/extract_libm_tables.py
"""
import glob
import os
import re
import struct
import sys
from pathlib import Path

import numpy as np

HDR = (Path(__file__).resolve().parent.parent / "paper_2605_08699_b200" / "csrc" /
       "libm_restated.cuh").read_text()


def header_doubles(name):
    m = re.search(name + r"\[\d+\] = \{(.*?)\};", HDR, re.S)
    return [float.fromhex(x.strip()) for x in m.group(1).split(",") if x.strip()]


def header_u64(name):
    m = re.search(name + r"\[\d+\] = \{(.*?)\};", HDR, re.S)
    return [int(x.strip().rstrip("ull"), 16) for x in m.group(1).split(",") if x.strip()]


def d(data, off):
    return struct.unpack("<d", data[off:off + 8])[0]


def main():
    so = glob.glob(os.path.dirname(np.__file__) + "/_core/_multiarray_umath*.so")[0]
    data = open(so, "rb").read()
    # exp8_ha: the 64-byte broadcast block holding the shift constant
    shift = struct.pack("<d", float.fromhex("0x1.8000000003ff0p+48")) * 8
    e = data.find(shift)
    base = e - 0x140
    t16 = [d(data, base + 8 * k) for k in range(16)]
    l16 = [d(data, base + 0x80 + 8 * k) for k in range(16)]
    ok = t16 == header_doubles("kSvExpT") and l16 == header_doubles("kSvExpL")
    print("svml exp8_ha tables", "match" if ok else "MISMATCH", hex(base))
    # log8_ha: the block with 1.0 then 0.75 broadcasts follows the two tables
    pat = struct.pack("<d", 1.0) * 8 + struct.pack("<d", 0.75) * 8
    ok2, lbase, lg = False, -1, data.find(pat)
    while lg >= 0 and not ok2:  # several SVML log variants share the prologue constants
        lbase = lg - 0x100
        lh = [d(data, lbase + 8 * k) for k in range(16)]
        ll = [d(data, lbase + 0x80 + 8 * k) for k in range(16)]
        ok2 = lh == header_doubles("kSvLogH") and ll == header_doubles("kSvLogL")
        lg = data.find(pat, lg + 1)
    print("svml log8_ha tables", "match" if ok2 else "MISMATCH", hex(lbase))
    libm = open("/lib/x86_64-linux-gnu/libm.so.6", "rb").read()
    h1 = struct.unpack("<Q", struct.pack("<d", 2 ** (1 / 128)))[0] - (1 << 45)
    i = libm.find(struct.pack("<Q", h1))
    tb = i - 24
    tab = [struct.unpack("<Q", libm[tb + 8 * k:tb + 8 * k + 8])[0] for k in range(256)]
    ok3 = tab == header_u64("kGlibcExpTab")
    print("glibc __exp_data.tab", "match" if ok3 else "MISMATCH", hex(tb))
    return 0 if (ok and ok2 and ok3) else 1


if __name__ == "__main__":
    sys.exit(main())
