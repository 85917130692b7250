cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/r02_syrkfuse_ab.log
for v in 1 0 1 0; do
  GBOPT_SYRK_FUSE=$v timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-sharded 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse=$v c4', round(d['ms_per_step'],3), round(d['value'],1), 'eval', round(d['roofline_eval']['frac_of_peak'],4), 'e2e', round(d['e2e']['value'],1), 'parity', d.get('parity'))" >> gpurun_out/r02_syrkfuse_ab.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_syrkfuse_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_syrkfuse_tests.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:nt_syrk_segs -c 1 -f -o gpurun_out/r02_ncu_syrkseg python tools/ncu_capture.py c4 > gpurun_out/r02_ncu_syrkseg.log 2>&1
