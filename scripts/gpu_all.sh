# tests + smoke + bench (+ reference arm) + ncu of the hot kernels, one GPU call.
TAG=${TAG:-rX}
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check_${TAG}.log 2>&1
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_${TAG}.log 2>&1
TAG=$TAG bash scripts/gpu_ncu.sh > gpurun_out/ncu_${TAG}.txt 2>&1
grep -E "passed|failed|smoke|value" gpurun_out/check_${TAG}.log | cut -c1-400
tail -1 gpurun_out/ref_${TAG}.log | cut -c1-300
tail -3 gpurun_out/ncu_${TAG}.txt | cut -c1-200
