# bench.py on every BASELINE config (c4 is the default line); one JSON line each
out=${1:-gpurun_out/bench_all.jsonl}
: > $out
for a in "--config c1" "--config c2" "--config c3" "--config c5 --rank 8" "--config c5 --rank 16" "--config c5 --rank 32" "--config c5 --rank 64" "--config c5 --rank 128" "--config c5 --rank 256" "--config c4"; do
  timeout 600 python bench.py $a --no-cpu-baseline >> $out 2>>${out%.jsonl}.err
done
