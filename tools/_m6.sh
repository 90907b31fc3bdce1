TED_PUSH=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "(two_gpus and peer and not stalled) or (four_gpus and peer and 2-2-1-8) or step_graph" > gpurun_out/m6_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/m6_tests.log; tail -2 gpurun_out/m6_tests.log
for rep in 1 2; do
for push in 1 0; do
 TED_PUSH=$push timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$rep$push bench.py --gpus 4 --steps 30 --warmup 5 --no-dtd-compare > gpurun_out/m6_b4_p${push}.log 2>&1
 grep '^{' gpurun_out/m6_b4_p${push}.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']
print('push=$push', round(d['ms_per_step'],3), 'e2e_ms', round(d['config']['tokens']/d['e2e']['value']*1e3,3), 'clk', d['clocks']['sm_mhz'], {k: s.get(k) for k in ['combine_pull','gate_dx','barrier','gemm2_fwd','dgrad1']})"
done; done
