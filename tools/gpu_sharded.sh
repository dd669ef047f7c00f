set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "sharded or small_segments" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-path sharded > gpurun_out/bs.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bs.log').read().strip().splitlines()[-1])
print('c1 sharded e2e', d['ms_per_step'], d['e2e'])" || tail -5 gpurun_out/bs.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bt1.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bt1.log').read().strip().splitlines()[-1])
print('torchrun n1', d['ms_per_step'], d['e2e'])" || tail -5 gpurun_out/bt1.log
