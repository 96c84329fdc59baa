# Reference arm (CPU) vs worker count on this box's host: the default (one per core, capped at 24) vs cores/2, cores/3.
n=$(python -c 'import os;print(os.cpu_count())'); echo "cpu_count=$n nproc=$(nproc)"; lscpu | grep -E "^CPU\(s\)|Thread|Core|Socket|Model name" | tr -s ' '
for w in 0 $((n/2)) $((n/3)) $((n/4)); do [ "$w" -lt 0 ] && continue
 echo "workers=$w $(timeout 600 python bench.py --impl reference --steps 2 --warmup 3 --cpu-workers $w 2>/dev/null | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());print("%.3g"%d["value"], d["cpu_baseline"]["sample"])')"
done
