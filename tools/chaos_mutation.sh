#!/bin/bash
# Does the race-stress comparison catch a real race? libktb_mut.so is the
# chaos build with S3's per-round block barrier removed (KTB_S3_ABL=4: the
# window RMW of one round then races the next round's). Built here with
#   KTB_LIB_NAME=libktb_mut.so KTB_EXTRA_FLAGS="-DKTB_CHAOS -DKTB_S3_ABL=4" \
#     python paper_2405_01599_b200/build.py
# Expected: tools/chaos_cases.py fails (S3 not reproducible / not equal).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/chaos_cases.py /tmp/ref.npz 3 > gpurun_out/chaos_mut_ref.log 2>&1
KTB_LIB_NAME=libktb_mut.so python tools/chaos_cases.py /tmp/mut.npz 6 > gpurun_out/chaos_mut.log 2>&1
echo "mutant exit code: $?" >> gpurun_out/chaos_mut.log
python - <<'PY' >> gpurun_out/chaos_mut.log 2>&1
import numpy as np, os
if os.path.exists("/tmp/mut.npz"):
    r, m = np.load("/tmp/ref.npz"), np.load("/tmp/mut.npz")
    for k in r.files:
        if k != "lib":
            print(k, "equal" if np.array_equal(r[k], m[k]) else "DIFFERS")
PY
tail -5 gpurun_out/chaos_mut.log
