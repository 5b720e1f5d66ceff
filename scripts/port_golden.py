"""Merges oracle-port slice values (gpurun_out/cfg5_oracle_<a>.npy, written on a GPU box
host by scripts/cfg5_parity.py) into tests/golden/cfg5_syc53_m20/port_single.bin (layout
of the reference's ref_*.bin: u64 n, u64 out_elems, u64 assignments[n], c128 values[n][out])
and its .json. usage: port_golden.py A [A ...]"""
import json
import os
import struct
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(REPO, "tests", "golden", "cfg5_syc53_m20")
b = open(os.path.join(D, "port_single.bin"), "rb").read()
n, oe = struct.unpack_from("<QQ", b, 0)
asg = list(np.frombuffer(b, np.uint64, n, 16))
vals = list(np.frombuffer(b, np.complex128, n * oe, 16 + 8 * n).reshape(n, oe))
for a in (int(x) for x in sys.argv[1:]):
    if a in [int(x) for x in asg]:
        continue
    v = np.load(os.path.join(REPO, "gpurun_out", f"cfg5_oracle_{a}.npy")).astype(np.complex128)
    asg.append(np.uint64(a))
    vals.append(v.ravel())
with open(os.path.join(D, "port_single.bin"), "wb") as f:
    f.write(struct.pack("<QQ", len(asg), oe))
    f.write(np.array(asg, np.uint64).tobytes())
    f.write(np.array(vals, np.complex128).tobytes())
meta_path = os.path.join(D, "port_single.json")
meta = json.load(open(meta_path))
meta["slices"] = len(asg)
meta["slice_digits"] = ("mixed radix of the assignments in port_single.bin (first sliced edge "
                        "most significant): " + ", ".join(str(int(x)) for x in asg))
json.dump(meta, open(meta_path, "w"), indent=1)
print(len(asg), [int(x) for x in asg])
