#!/bin/bash
# per-kernel table from an ncu report
ncu -i "$1" --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.sum,launch__grid_size,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]; u=rows[1]
def f(r,k):
    return r[h.index(k)]
print('%-28s %9s %9s %9s %6s %6s %6s %5s %10s %6s' % ('kernel','us','dramMB','GB/s','sm%','mem%','warp%','regs','Minst','L2hit'))
for r in rows[2:]:
    n=f(r,'Kernel Name').split('(')[0].split('::')[-1][:28]
    t=float(f(r,'gpu__time_duration.sum'))
    tu=u[h.index('gpu__time_duration.sum')]
    if tu=='ms': t*=1000
    if tu=='ns': t/=1000
    def mb(k):
        v=float(f(r,k)); un=u[h.index(k)]
        return v*{'Gbyte':1000,'Mbyte':1,'Kbyte':1e-3,'byte':1e-6}[un]
    d=mb('dram__bytes_read.sum')+mb('dram__bytes_write.sum')
    print('%-28s %9.1f %9.1f %9.0f %6.1f %6.1f %6.1f %5s %10.2f %6.1f' % (n,t,d,d/t*1e3 if t else 0,float(f(r,'sm__throughput.avg.pct_of_peak_sustained_elapsed')),float(f(r,'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed')),float(f(r,'sm__warps_active.avg.pct_of_peak_sustained_active')),f(r,'launch__registers_per_thread'),float(f(r,'smsp__inst_executed.sum'))/1e6,float(f(r,'lts__t_sector_hit_rate.pct'))))
"
