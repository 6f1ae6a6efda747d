for V in 1024 512; do export FS_PERSIST_BLOCK=$V; echo "== block $V"; python scripts/ens_phases.py 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:persist --csv python scripts/prof_ens.py 2>/dev/null | grep persist | awk -F'","' '{gsub(/"/,"",$15); s+=$15; n++} END {print "persist launches", n, "mean us", s/n/1000}'
done
