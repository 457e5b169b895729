mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe tools/dmma_probe.cu && /tmp/dmma_probe > gpurun_out/dmma_probe.txt 2>&1
for v in seg_base seg_v1; do echo "== $v"; DOT_LIB_PATH=$PWD/paper_1706_05586_b200/lib/variants/$v.so timeout 600 python tools/seg_bench.py full64 all128; done > gpurun_out/seg_bench.txt 2>&1
cat > /tmp/mm.py <<'P'
import torch
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn_like(a)
for _ in range(3): c=a@b
torch.cuda.synchronize()
P
timeout 300 ncu --metrics launch__registers_per_thread,launch__block_size,launch__grid_size,launch__shared_mem_per_block_dynamic,launch__cluster_dim_x,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__warps_active.avg.per_cycle_active,gpu__time_duration.sum -c 2 python /tmp/mm.py > gpurun_out/ncu_dgemm.txt 2>&1
cat gpurun_out/dmma_probe.txt gpurun_out/seg_bench.txt; grep -E "gemm|Kernel|registers|block_size|grid_size|shared_mem|dmma|warps_active|duration|cluster" gpurun_out/ncu_dgemm.txt | head -40
