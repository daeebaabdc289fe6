#!/bin/bash
# Same-box A/B: time the kinds given ($@, default asm) with libskgpu_base.so
# (tools/ab_build.sh: HEAD) and the working tree's libskgpu.so, interleaved.
# AB_TESTS=1 runs the asm + parity GPU tests on the working tree first.
cd "$(dirname "$0")/.."
kinds=${@:-asm}
[ -n "$AB_TESTS" ] && timeout 900 python -m pytest tests/test_gpu_asm.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for r in 1 2; do
  for lib in base ""; do
    for k in $kinds; do
      echo -n "${lib:-new} "
      SKGPU_LIB=paper_2305_09493_b200/libskgpu${lib:+_$lib}.so python tools/prof_disasm.py --modules 200000 --kind $k
    done
  done
done
