# A/B of library builds on the same box: stage times of cfg2/cfg4/cfg5 (tools/time_cpqr.py), alternating.
# usage: bash tools/ab_lib.sh base new [rounds]   (paper_2105_07076_b200/ab/<name>.so; "pkg" = the package library)
A=${1:-base}; B=${2:-pkg}; R=${3:-2}
lib() { if [ "$1" = "pkg" ]; then echo paper_2105_07076_b200/libidkit_b200.so; else echo paper_2105_07076_b200/ab/$1.so; fi; }
for r in $(seq 1 $R); do for v in $A $B; do for c in cfg4 cfg5 cfg2; do
  IDK_LIB_PATH=$(lib $v) python tools/time_cpqr.py $c 10 2>/dev/null | sed "s/^/$v: /"
done; done; done
