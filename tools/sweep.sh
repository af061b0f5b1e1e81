# usage inside gpurun: bash tools/sweep.sh "-DFOO=1" "-DFOO=2" ...
# per variant: rebuild, quick parity (reference 1080p golden, goldens with forced
# launch variants, ragged batches), then the cfg4 bench line's key kernels
for flags in "$@"; do
  FVV_NVCC_EXTRA="$flags" python -c "from paper_2112_10603_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || { echo "$flags BUILD FAILED"; continue; }
  python -m pytest tests/test_gpu_timed_path.py -q -x -p no:cacheprovider -k "reference_golden or forced or assemble" > gpurun_out/sw_t.log 2>&1
  par=$(tail -1 gpurun_out/sw_t.log)
  python bench.py --cpu-budget 1 --no-vinet --steps 20 > gpurun_out/sw.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms_per_step']; print(sys.argv[1], '|', sys.argv[2], '|', round(d['value']), {a:b for a,b in k.items() if a in ('k_sad<0>','k_sad<1>','k_sad<2>','k_mask_cols','k_blend','k_warpq<2>','k_scan_carry')})" "$flags" "$par" | tee -a gpurun_out/sweep_results.log
done
