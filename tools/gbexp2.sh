cat > /tmp/gbrun.py <<'PY'
import sys; sys.path.insert(0,".")
import synth
from paper_1410_0562_b200 import SetBWTE
d,o=synth.uniform(3000000,100,seed=1)
ix=SetBWTE("ACGT",block_suffixes=1<<27); ix.set_option("gather_buckets",1); ix.append(d,o); ix.append(d,o)
PY
for v in 0 1; do
if [ $v = 1 ]; then export SETBWTE_GB_SIMPLE=1; fi
ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gb_fetch -s 3 -c 1 --csv --log-file gpurun_out/gbexp2_$v.csv python /tmp/gbrun.py > /dev/null 2>&1
done
