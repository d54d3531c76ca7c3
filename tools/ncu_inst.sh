# instruction counts and durations of every kernel of one c3 frame (dev tool)
# usage: bash tools/ncu_inst.sh ["ENV=.. ENV2=.."]...
for c in "${@:-}"; do
  echo "== $c"
  env $c ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__thread_inst_executed.sum --clock-control none -s 15 -c 5 --csv python tools/quick_timing.py 2>/dev/null | grep -E "_kernel" | awk -F'","' '{split($5,k,"("); print k[1], $(NF-2), $NF}' | sed 's/"//g'
done
