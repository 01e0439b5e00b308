# dev: Gram kernel time + DRAM traffic at config 5 (with and without the G stores)
timeout 100 python scripts/timing_probe.py 5 2>&1 | tail -1
timeout 100 python scripts/screen_probe.py 2>&1 | tail -1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:syrk -s 1 -c 1 python scripts/timing_probe.py 5 2>&1 | grep -E "duration|bytes|sectors"
timeout 300 ncu --metrics $M --clock-control none -k regex:syrk -s 1 -c 1 python scripts/screen_probe.py 2>&1 | grep -E "duration|bytes|sectors"
