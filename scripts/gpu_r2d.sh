export NCCL_DEBUG=WARN
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
timeout 900 $TR scripts/ddp_check.py > gpurun_out/r2d_ddp_check.log 2>&1; echo "ddp_check rc=$?"
grep -E "OK|FAIL|PASSED|FAILED|Error|error" gpurun_out/r2d_ddp_check.log | head -40
for mode in "" "--zero1" "--grad-bf16" "--zero1 --grad-bf16"; do
  tag=$(echo "$mode" | tr -d ' -'); [ -z "$tag" ] && tag=ddp
  timeout 600 $TR bench.py --gpus 2 --steps 10 --warmup 3 $mode > gpurun_out/r2d_bench650_n2_$tag.json 2> gpurun_out/r2d_bench650_n2_$tag.err
  echo "bench $tag rc=$?"; python -c "import json,sys; d=json.loads(open('gpurun_out/r2d_bench650_n2_$tag.json').read().strip().splitlines()[-1]); print('$tag', d['value'], d['ms_per_step'], d['mfu'], d['config']['parallelism'], d['config']['cuda_graph'], d['kernels'].get('esm_adamw'), d['kernels'].get('esm_adamw_bf16g'))" || tail -20 gpurun_out/r2d_bench650_n2_$tag.err
done
