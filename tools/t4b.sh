set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py tests/test_gpu_fullsize.py -q -x -k "solve or lu or 4b" -p no:cacheprovider > gpurun_out/t4b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4b_pytest.log
for v in nopiv shift; do
  LM_BATCHED_LU=$v timeout 300 python bench.py --config 4b --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/t4b_$v.json 2> gpurun_out/t4b_$v.err
done
tail -3 gpurun_out/t4b_pytest.log
for v in nopiv shift; do python -c "
import json,sys; d=json.load(open('gpurun_out/t4b_$v.json')); print('$v', d['ms_per_step'], d['roofline'], d.get('verified'))"; done
