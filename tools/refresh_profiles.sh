# Round-end evidence refresh (run under gpurun): GPU tests, smoke, bench lines for every
# config, the cfg4 SAD-path launch list and the VINet rig-frame launch list.
TAG=${TAG:-r2_v1}
python -m pytest tests -q -m gpu 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for c in cfg4 cfg1 cfg2 cfg3 cfg5; do
  python bench.py --config $c > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
done
NOSIDE="--no-vinet --no-direct --no-encoder"
python bench.py --steps 2 --warmup 1 $NOSIDE --cpu-budget 1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/${TAG}_cfg4_launches.csv \
      python bench.py --steps 2 --warmup 1 $NOSIDE --cpu-budget 1 > /dev/null 2>&1
python tools/vinet_bench.py 1920 1080 7 rig2 && \
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file gpurun_out/${TAG}_vinet_launches.csv \
      python tools/vinet_bench.py 1920 1080 7 rig2 > /dev/null 2>&1
ls gpurun_out/${TAG}_*
