# usage inside gpurun: bash sweep.sh "-DFOO=1" "-DFOO=2" ...
for flags in "$@"; do
  FVV_NVCC_EXTRA="$flags" python -c "from paper_2112_10603_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
  python bench.py --cpu-budget 1 --no-vinet > gpurun_out/sw.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); k=d['roofline']['per_kernel_ms_per_step']; print(sys.argv[1], round(d['value']), {a:b for a,b in k.items() if a in ('k_sad<0>','k_sad<1>','k_sad<2>','k_mask_cols','k_blend','k_warpq<2>')})" "$flags"
done
