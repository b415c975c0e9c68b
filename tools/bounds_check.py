"""Cross-check of tools/bounds.cu's rates (dev aid): prints the rates for the c2 shape."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import __graft_entry__
    lib = ctypes.CDLL(__graft_entry__.build_bounds())
    lib.bounds_mix.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.POINTER(ctypes.c_double)]
    out = {}
    for ng, nr in ((3, 2), (3, 0), (0, 2), (1, 1), (2, 1), (5, 3)):
        u = ctypes.c_double()
        rc = lib.bounds_mix(128, 12_800_000, 12_800_000, ng, nr, 5, ctypes.byref(u))
        out[f"{ng}g{nr}r"] = {"rc": rc, "units_per_s": u.value, "ms_per_10M_units": 1e7 / u.value * 1e3 if u.value else None}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
