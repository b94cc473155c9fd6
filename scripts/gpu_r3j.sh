# 3B per-GPU batch (4 / 8 / 12 x 1024) and the 650M batch (16 / 24 x 1024) at one B200
mkdir -p gpurun_out
for b in 4 8 12; do
  timeout 900 python bench.py --config 3b --batch $b --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3j_b.json 2> gpurun_out/r3j_b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3j_b.json').read().strip().splitlines()[-1]); print('3b B=$b', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r3j_b.err
done
for b in 16 24; do
  timeout 900 python bench.py --config 650m --batch $b --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3j_b.json 2> gpurun_out/r3j_b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r3j_b.json').read().strip().splitlines()[-1]); print('650m B=$b', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r3j_b.err
done
