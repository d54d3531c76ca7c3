for c in "" "STEREO_POST_ROWS=4" "STEREO_POST_ROWS=8" "STEREO_POST_ROWS=4 STEREO_POST_THREADS=256"; do
  echo "== $c"
  env $c ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__thread_inst_executed.sum --clock-control none -k regex:"sd_|prep|post" -s 15 -c 3 --csv python tools/quick_timing.py 2>/dev/null | grep -E "sd_|prep|post" | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
done
