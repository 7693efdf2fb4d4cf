# Reference-schema benchmark reports, GPU drop-in vs reference CPU (one GPU call).
OUT=${OUT:-gpurun_out/reports}
mkdir -p $OUT
B=scripts/refbench/_build
for impl in b200 reference; do
  for mode in cfar pipeline; do
    for fmt in text json csv; do
      timeout -s KILL 600 $B/refbench_$impl $mode $fmt 10 > $OUT/${mode}_${impl}.$fmt 2> $OUT/${mode}_${impl}.$fmt.err
    done
  done
done
cat $OUT/cfar_b200.text $OUT/cfar_reference.text $OUT/pipeline_b200.text $OUT/pipeline_reference.text
