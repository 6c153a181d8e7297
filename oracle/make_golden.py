#!/usr/bin/env python3
"""TEST INFRASTRUCTURE (oracle) — regenerates the committed golden fixtures.

Runs oracle/_ref/golden_dump (the UNMODIFIED reference headers from
/root/reference/proj/include compiled with the strict Eigen shim, see
oracle/Makefile) and converts its tagged binary output into
tests/golden/<scenario>.npz.  Only needed in the build container, where
/root/reference exists; the .npz files are committed and travel.

    python oracle/make_golden.py            # all scenarios
    python oracle/make_golden.py rng plan   # a subset
"""
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
DTYPES = {0: np.float32, 1: np.float64, 2: np.uint32, 3: np.uint64,
          4: np.int32, 5: np.int64, 6: np.uint8}
SCENARIOS = ["rng", "plan", "synth", "nn", "surrogate", "trainer", "tournament", "outputs",
             "horizon", "tournament_paper", "activations"]
RUN_DIRS = ["run_tiny_k2", "run_tiny_single"]  # written by the "outputs" scenario


def read_tagged(path):
    out = {}
    with open(path, "rb") as f:
        buf = f.read()
    pos = 0
    while pos < len(buf):
        (nlen,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        name = buf[pos:pos + nlen].decode()
        pos += nlen
        code = buf[pos]
        pos += 1
        (count,) = struct.unpack_from("<Q", buf, pos)
        pos += 8
        dt = np.dtype(DTYPES[code]).newbyteorder("<")
        nbytes = count * dt.itemsize
        out[name] = np.frombuffer(buf, dtype=dt, count=count, offset=pos).copy()
        pos += nbytes
    return out


def main(argv):
    want = argv or SCENARIOS
    subprocess.check_call(["make", "-C", HERE, "_ref/golden_dump"])
    with tempfile.TemporaryDirectory() as raw, tempfile.TemporaryDirectory() as tmp:
        subprocess.check_call([os.path.join(HERE, "_ref", "golden_dump"), raw, tmp] + want)
        os.makedirs(os.path.join(REPO, "tests", "golden"), exist_ok=True)
        for s in want:
            arrays = read_tagged(os.path.join(raw, s + ".bin"))
            dst = os.path.join(REPO, "tests", "golden", s + ".npz")
            np.savez_compressed(dst, **arrays)
            print(f"{dst}: {len(arrays)} arrays, {os.path.getsize(dst)} bytes")
        if "outputs" in want:  # reference run directories, copied verbatim
            import shutil
            for rd in RUN_DIRS:
                dst = os.path.join(REPO, "tests", "golden", rd)
                shutil.rmtree(dst, ignore_errors=True)
                shutil.copytree(os.path.join(raw, rd), dst)
                print(f"{dst}: {sorted(os.listdir(dst))}")
            # one bundle file the reference's ensure_dataset wrote (LBDS bytes)
            shutil.copy(os.path.join(tmp, "data_tiny_k2", "bundle_00000.lbds"),
                        os.path.join(REPO, "tests", "golden", "run_tiny_k2_bundle_00000.lbds"))
            subprocess.check_call(["make", "-C", HERE, "_ref/nl_doubles"])
            dst = os.path.join(REPO, "tests", "golden", "nlohmann_doubles.txt")
            with open(dst, "w") as f:
                subprocess.check_call([os.path.join(HERE, "_ref", "nl_doubles"), "4000"], stdout=f)
            print(f"{dst}: {os.path.getsize(dst)} bytes")


if __name__ == "__main__":
    main(sys.argv[1:])
