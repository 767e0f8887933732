for v in pkg $*; do
  if [ "$v" = "pkg" ]; then L=paper_2105_07076_b200/libidkit_b200.so; else L=paper_2105_07076_b200/ab/$v.so; fi
  for a in "20000 16" "30000 16" "24000 16" "16000 16 50000" "8000 32"; do
    IDK_LIB_PATH=$L timeout 300 python tools/time_streaming.py $a 2>&1 | tail -1 | cut -c1-100 | sed "s/^/$v: /"
  done
done
