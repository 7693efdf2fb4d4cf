# end-of-round measurement set (one GPU call)
TAG=${TAG:-rX}
export PYTHONPATH=.
mkdir -p gpurun_out
TAG=$TAG bash scripts/gpu_all.sh
python bench.py --fused --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fused_${TAG}.log 2>&1
TAG=${TAG}f MAPS=4096 KREGEX=cfar_fused KSKIP=1 KCOUNT=1 CMDX=--fused bash scripts/gpu_ncu.sh > gpurun_out/ncuf_${TAG}.txt 2>&1
for c in 1 2 4 5 6; do timeout -s KILL 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/cfg${c}_${TAG}.log 2>&1; done
tail -1 gpurun_out/fused_${TAG}.log | cut -c1-400
for c in 1 2 4 5 6; do tail -1 gpurun_out/cfg${c}_${TAG}.log | cut -c1-300; done
