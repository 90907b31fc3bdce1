for rep in 1 2; do
for push in 1 0; do for graph in 1 0; do
 TED_PUSH=$push TED_GRAPH=$graph timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$rep$push$graph bench.py --gpus 4 --steps 30 --warmup 5 --no-dtd-compare > gpurun_out/m5_b4_p${push}_g${graph}.log 2>&1
 grep '^{' gpurun_out/m5_b4_p${push}_g${graph}.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms']
print('push=$push graph=$graph', round(d['ms_per_step'],3), 'e2e_ms', round(d['config']['tokens']/d['e2e']['value']*1e3,3), 'clk', d['clocks']['sm_mhz'], {k: s.get(k) for k in ['combine_pull','gate_dx','barrier','gemm2_fwd','dgrad1']})"
done; done; done
