# usage inside gpurun: [CONFIGS="cfg4 cfg2"] bash tools/sweep_scan.sh "-DFOO=1" ...
# per variant: rebuild, GPU parity tests, bench (SAD path) on each config
for flags in "$@"; do
  FVV_NVCC_EXTRA="$flags" python -c "from paper_2112_10603_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  t=$(python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1)
  for c in ${CONFIGS:-cfg4}; do
    python bench.py --config $c --cpu-budget 1 --no-vinet > gpurun_out/sw.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms_per_step']; print(sys.argv[1], sys.argv[3], sys.argv[2], round(d['value']), round(d['ms_per_step'],3), {a:b for a,b in k.items() if a in ('k_scan_carry','k_blend','k_mask_cols')})" "$flags" "$t" "$c"
  done
done
