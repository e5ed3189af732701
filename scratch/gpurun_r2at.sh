mkdir -p gpurun_out
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-fasterpam --no-dissimilarity --no-cpu-baseline --no-clara"
timeout 900 ncu --cache-control none --clock-control none -k regex:"k_fp1_post|k_swap_stream_seg2" -s 6 -c 4 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --csv $CMD > gpurun_out/r2at_ncu_nocache.csv 2> gpurun_out/r2at_ncu.err; echo rc=$?
