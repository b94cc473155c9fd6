# cost of dropout: Geneformer with BERT's 0.02 / 0.02 (hidden, attention) vs none; 650M with attention dropout 0.1
mkdir -p gpurun_out
for spec in "geneformer 0,0" "geneformer 0.02,0.02" "geneformer 0,0.02" "650m 0,0.1"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --dropout $2 --no-cpu-baseline --no-e2e > gpurun_out/r4e_$1_$2.json 2> gpurun_out/r4e_$1_$2.err
  python -c "
import json; d=json.loads(open('gpurun_out/r4e_$1_$2.json').read().strip().splitlines()[-1]); k=d['kernels']
print('$1 dropout=$2', round(d['value']), round(d['ms_per_step'],2), d['mfu'], d['clocks']['sm_mhz'], d['loss'], {n: (v['ms'], v['launches']) for n, v in k.items() if 'attn' in n})" || tail -5 gpurun_out/r4e_$1_$2.err
done
