# One bench line per BASELINE config and per word width (C2 shape).
set -x
rm -f gpurun_out/bench_all.jsonl gpurun_out/bench_all.err
python __graft_entry__.py > /dev/null 2>&1
for cfg in c1 c2 c3 c4 c4seg c3cat; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --cpu-min-time 2 >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; echo $cfg=$?
done
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --cpu-min-time 2 >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; echo c5=$?
for w in 16 32 64; do
  timeout 600 python bench.py --config c2 --width $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; echo w$w=$?
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; echo torchrun1=$?
timeout 300 python bench.py --impl reference >> gpurun_out/bench_all.jsonl 2>> gpurun_out/bench_all.err; echo ref=$?
tail -5 gpurun_out/bench_all.err
