#!/bin/bash
# Development build with the sweep kernel's per-phase cycle counters (-DSPMESL_TAIL_PROF) into
# scripts/_prof/libspmesl.so (not the shipped library).  Run from the repo root.
set -e
D=scripts/_prof; mkdir -p $D
python - <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
import paper_2203_15031_b200.build as b
D = "scripts/_prof"
objs = []
for src in b.SOURCES:
    obj = os.path.join(D, src + ".o"); objs.append(obj)
    flags = b.FLAGS + (["-DSPMESL_TAIL_PROF"] if src == "tail.cu" else [])
    src_path = os.path.join(b.CSRC, src)
    if src != "tail.cu" and os.path.exists(os.path.join(b.BUILD, src + ".o")):
        subprocess.run(["cp", os.path.join(b.BUILD, src + ".o"), obj], check=True); continue
    subprocess.run([b.NVCC] + b.ARCH + flags + ["-c", src_path, "-o", obj], check=True, capture_output=True)
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", os.path.join(D, "libspmesl.so")] + objs +
               ["-lcudart_static", "-lrt", "-lpthread", "-ldl"], check=True)
print(os.path.join(D, "libspmesl.so"))
PY
