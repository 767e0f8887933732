# A/B of two library builds on the same box (IDK_LIB_PATH), alternating: CPQR step times
# Build the variants first, e.g. paper_2105_07076_b200/ab/A.so and B.so (the package .so linked with a
# different cpqr_resident.o), then: gpurun -- bash tools/ab_cpqr.sh
for r in 1 2; do for v in A B; do
  for c in cfg2 cfg4; do IDK_LIB_PATH=paper_2105_07076_b200/ab/$v.so python tools/trace_cpqr.py $c 2>/dev/null | grep "step (cta0)" | sed "s/^/$v $c: /"; done
done; done
