OUT=gpurun_out
python tools/bench_layers.py --suite mobilenet --batch 128 --reps 3 > $OUT/bw_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  -k regex:"dw3_tma|depthwise|requantize|quantize|dequantize" --csv --log-file $OUT/bw_launches.csv \
  python tools/bench_layers.py --suite mobilenet --batch 128 --reps 3 > $OUT/ncu_bw.log 2>&1
echo "bw rc=$?"
python tools/bench_layers.py --suite requant --reps 3 > $OUT/rq_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  -k regex:"requantize|quantize|dequantize" --csv --log-file $OUT/rq_launches.csv \
  python tools/bench_layers.py --suite requant --reps 3 > $OUT/ncu_rq.log 2>&1
echo "rq rc=$?"
