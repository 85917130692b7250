cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_gputest.log
python -m pytest tests/test_gpu_ref_parity.py -q -s -p no:cacheprovider -k full_size > gpurun_out/r02_refparity.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
