# PWLS kernels: parity + vector/scalar agreement, 256^3 HBM kernel table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pwls.py tests/test_gpu_recon.py tests/test_gpu_subsets.py -q -x > gpurun_out/r26_tests.log 2>&1; echo "TESTS EXIT $?"; tail -3 gpurun_out/r26_tests.log
timeout 900 python tools/hbm_kernels.py > gpurun_out/hbm_r26.json 2> gpurun_out/hbm_r26.err; echo "HBM EXIT $?"
python -c "
import json;d=json.load(open('gpurun_out/hbm_r26.json'))
for k,v in d['kernels'].items(): print('%-26s %8.1f us %6.0f GB/s %.2f'%(k,v['us'],v['gbs'],v['frac_measured']))"
