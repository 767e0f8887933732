# A/B of two library builds on the same box (IDK_LIB_PATH), alternating: CPQR step times.
# Build the variants first, e.g. paper_2105_07076_b200/ab/A.so and B.so (the package .so linked with a
# different cpqr_resident.o), then: gpurun -- bash tools/ab_cpqr.sh
IDK_LIB_PATH=paper_2105_07076_b200/ab/B.so python -m pytest tests -x -q -m gpu -k "qr or id or rid or config or edge" 2>&1 | tail -1
for r in 1 2; do for v in A B; do
  for c in cfg2 cfg4 cfg5; do IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python tools/trace_cpqr.py $c 2>/dev/null | grep "step (cta0)" | sed "s/^/$v $c: /"; done
done; done
