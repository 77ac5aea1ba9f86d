mkdir -p gpurun_out/w2rep
for i in 1 2 3 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2971$i bench.py --gpus 2 --no-cpu-baseline > gpurun_out/w2rep/w2_$i.json 2>/dev/null
done
for f in gpurun_out/w2rep/*.json; do python -c "
import json,sys
l=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', l['ms_per_step'], l['host_enqueue_us_per_step'])"; done
