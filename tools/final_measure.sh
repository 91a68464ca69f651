set -x
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-decode --no-parity"
timeout 300 $B > gpurun_out/pre.json 2>&1 || exit 1
timeout 900 ncu --clock-control none --kernel-name-base demangled -k regex:stpc:: --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.avg.per_cycle_active,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/stages.csv $B > gpurun_out/ncu_stages.log 2>&1
python tools/ncu_stages.py gpurun_out/stages.csv profiles/r2_ncu_stages.json && cp profiles/r2_ncu_stages.json gpurun_out/
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 ncu --kernel-name-base mangled -k regex:_ZN4stpc --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-parity --decode-e2e-groups 8 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"convert_staged|fit_pair|emit_residual_compact|start_tiles_staged|refit_all" -c 7 -o gpurun_out/final_full $B > gpurun_out/ncu_full.log 2>&1
timeout 300 python tools/latency_table.py > gpurun_out/lat_final.txt 2>&1
echo done
