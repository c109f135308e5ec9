# Config 5 throughput sweep over N (BASELINE.json config 5: N = 2^14 .. 2^20),
# one bench line per size and rule; run on a GPU box from the repo root.
mkdir -p gpurun_out; rm -f gpurun_out/c5_sizes.jsonl
for n in 16384 65536 262144 1048576; do
  r=$(( n >= 262144 ? 100 : 400 ))
  timeout 300 python bench.py --no-cpu-baseline --n $n --rounds $r --steps 5 2>&1 | tail -1 >> gpurun_out/c5_sizes.jsonl
done
