# K3 tensor-pipe / L2 metrics at fc1, fc2, cfg1 and on the INT8 peak probe
# (the probe calibrates what 100% MMA issue reads as), plus one --set full
# capture of K3 at fc1.  OUT=<name> bash tools/gpu_k3ncu.sh
OUT=gpurun_out/${OUT:-r02k3}; mkdir -p $OUT
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_imma.sum,sm__inst_executed_pipe_tc.sum,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for s in "4608 3072 12288" "4608 12288 3072" "4096 3072 3072" "4608 3072 3072"; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:k3_v4 -s 2 -c 1 --csv python tools/k3_one.py $s 3 > $OUT/k3_metrics_${s// /_}.csv 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -k regex:mma_loop -s 1 -c 4 --csv ./tools/probes/i8_peak_probe > $OUT/probe_metrics.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_v4 -s 2 -c 1 -o $OUT/k3_fc1 python tools/k3_one.py 4608 3072 12288 3 > $OUT/ncu_full.log 2>&1
python tools/k3_time.py > $OUT/k3_time.txt 2>&1
tail -3 $OUT/ncu_full.log; cat $OUT/k3_time.txt; ls $OUT
