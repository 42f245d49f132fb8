"""Generate golden vectors from the REFERENCE's own code (oracle/_ref/libfgfrft_ref_shim.so,
compiled by oracle/Makefile from /root/reference/proj/include/fgfrft/{sinc,rng}.hpp).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The JSON files are committed so tests run without /root/reference (e.g. on the GPU box).
Doubles are stored as float.hex() strings: bit-exact round trip.
"""
import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"])
    ref = ctypes.CDLL(os.path.join(ROOT, "oracle", "_ref", "libfgfrft_ref_shim.so"))
    ref.ref_sinc_coeffs.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    ref.ref_sinc_coeffs.restype = ctypes.c_int
    ref.ref_fnv1a64.restype = ctypes.c_uint64
    ref.ref_fnv1a64.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    ref.ref_rng_derive.restype = ctypes.c_uint64
    ref.ref_rng_derive.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    ref.ref_rng_stream.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]

    # sinc coefficients: the orders of test_sinc.cpp / test_transform.cpp / acceptance.cpp and
    # the BASELINE configs (alpha = 0.37, the config-2 sweep endpoints and interior points).
    cases = []
    alphas = [0.0, 1.0, -3.0, 0.5, 0.15, 0.35, 0.55, 0.75, 0.95, 1.3, -0.4, 2.7, 0.3, -0.3, 1.0000004,
              -1.0000004, 2.5, -2.5, 1e-8, -1e-8, 7.3, -7.3, 0.37, 0.7, 1.5, 2.2, 9.0, 5e-7, 2e-6,
              1.0 + 3e-5, -2.0 - 3e-5] + list(np.linspace(0.0, 2.0, 64))
    for a in alphas:
        for l in (2, 6, 8, 10, 16, 32, 64, 128):
            c = np.empty(2 * l + 1)
            dc = np.empty(2 * l + 1)
            assert ref.ref_sinc_coeffs(a, l, c.ctypes.data, dc.ctypes.data) == 0
            cases.append({"alpha": float(a).hex(), "l": l, "c": [float(v).hex() for v in c],
                          "dc": [float(v).hex() for v in dc]})
    with open(os.path.join(HERE, "sinc_coeffs.json"), "w") as fh:
        json.dump({"source": "reference sinc.hpp:50-63 via oracle/_ref", "cases": cases}, fh)

    # RNG streams (rng.hpp:12-56): interleaved uniform/gaussian draws for several seeds.
    streams = []
    for seed in (0, 1, 7, 42, 0xDEADBEEF, 2**63 + 5):
        kinds = np.random.default_rng(seed % 2**32).integers(0, 2, 257).astype(np.int32)
        out = np.empty(257)
        ref.ref_rng_stream(ctypes.c_uint64(seed), kinds.ctypes.data, 257, out.ctypes.data)
        streams.append({"seed": str(seed), "kinds": kinds.tolist(), "values": [float(v).hex() for v in out]})
    derive = [{"seed": str(s), "index": str(i), "value": str(ref.ref_rng_derive(s, i))}
              for s in (0, 1, 42, 2**64 - 1) for i in (0, 1, 2, 1000, 4095)]
    with open(os.path.join(HERE, "rng_stream.json"), "w") as fh:
        json.dump({"source": "reference rng.hpp:12-56 via oracle/_ref", "streams": streams, "derive": derive}, fh)

    # FNV-1a fingerprints (rng.hpp:59-67) of deterministic byte buffers.
    fnv = []
    for n in (0, 1, 7, 16, 1000, 65536):
        buf = (np.arange(n, dtype=np.uint64) * 2654435761 % 251).astype(np.uint8)
        fnv.append({"n": n, "value": str(ref.ref_fnv1a64(buf.ctypes.data, n))})
    with open(os.path.join(HERE, "fnv1a64.json"), "w") as fh:
        json.dump({"source": "reference rng.hpp:59-67 via oracle/_ref",
                   "buffer": "bytes[i] = (i * 2654435761) % 251", "cases": fnv}, fh)
    print("golden vectors written")


if __name__ == "__main__":
    main()
