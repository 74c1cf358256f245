# A/B of library variants on a probe config: bash tools/r2_ab.sh "<probe args>" default u1 u2np ...
args=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=paper_1701_05975_b200/lib_var/libwbc_$v.so; fi
  echo "== $v"
  WBC_LIB=$lib timeout 600 python tools/probe_perf.py $args 2>&1 | grep -E "^rep|phase share|per source" | tail -3
done
