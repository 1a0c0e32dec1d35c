"""Regenerates tests/golden/rng_streams.json from the reference's own rng.hpp.

oracle/_ref/rng_golden is built by `make -C oracle ref` straight from
/root/reference/proj/include/isnmf/rng.hpp (this container only; the reference
is not on the GPU box).  The JSON it prints is committed as the golden fixture.
usage: python tests/golden/gen_rng_golden.py
"""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "rng_golden")], check=True, capture_output=True,
                     text=True).stdout
data = json.loads(out)
data["_source"] = ("printed by oracle/_ref/rng_golden = oracle/ref/rng_golden.cpp compiled against "
                   "/root/reference/proj/include/isnmf/rng.hpp (rng.hpp:10-44; online.hpp:79-87, 294-301; "
                   "test_kernels.cpp:13-19)")
with open(os.path.join(HERE, "rng_streams.json"), "w") as f:
    json.dump(data, f, indent=1)
print("wrote", os.path.join(HERE, "rng_streams.json"))
