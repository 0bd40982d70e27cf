for sh in 23 21 20; do
SETBWTE_GB_SHIFT=$sh ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:gb_fetch -s 2 -c 1 --csv --log-file gpurun_out/r2_gbexp_$sh.csv python tools/run_once.py --reads 20000000 --M 134217728 > /dev/null 2>&1
done
