export NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT NCCL_DEBUG_FILE=/tmp/nprobe.%h.%p.log
python -c "
import torch
from paper_2405_01599_b200 import dist as D
c = D.Comm.nccl(device=0)
print('made', c.world)
" > gpurun_out/nprobe.out 2>&1
ls -la /tmp/ | grep -i nprobe >> gpurun_out/nprobe.out
cat /tmp/nprobe* >> gpurun_out/nprobe.out 2>&1
unset NCCL_DEBUG_FILE
python -c "
import torch
from paper_2405_01599_b200 import dist as D
c = D.Comm.nccl(device=0)
" >> gpurun_out/nprobe.out 2>&1
