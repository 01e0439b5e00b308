#!/bin/bash
# Development: build libspmesl.so with tail.cu compiled under extra -D flags into
# scripts/_var/<name>/ (gitignored; travels to the GPU box).  Usage: build_variant.sh name "-DX=1 ..."
set -e
NAME=$1; shift
D=scripts/_var/$NAME; mkdir -p $D
python - "$D" "$@" <<'PY'
import os, subprocess, sys
sys.path.insert(0, ".")
import paper_2203_15031_b200.build as b
D, extra = sys.argv[1], sys.argv[2].split() if len(sys.argv) > 2 else []
b.build()
objs = []
for src in b.SOURCES:
    obj = os.path.join(b.BUILD, src + ".o")
    if src == "tail.cu":
        obj = os.path.join(D, "tail.cu.o")
        subprocess.run([b.NVCC] + b.ARCH + b.FLAGS + extra + ["-c", os.path.join(b.CSRC, src), "-o", obj],
                       check=True, capture_output=True)
    objs.append(obj)
subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-o", os.path.join(D, "libspmesl.so")] + objs +
               ["-lcudart_static", "-lrt", "-lpthread", "-ldl"], check=True)
print(os.path.join(D, "libspmesl.so"))
PY
