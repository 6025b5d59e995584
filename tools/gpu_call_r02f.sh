#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 300 python tools/oz_diag.py > gpurun_out/oz_diag.log 2>&1
TCB_OZAKI=0 timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2107_01384_b200 as tcb, synth
x = synth.grf_torch(n=1024, kmax=341, seed=0)
r = tcb.compress_device(x.data_ptr(), x.numel() * 4, tcb.Dtype.float32, list(x.shape), tcb.Params(target_re=1e-2))
print('c5 dmma: ranks', r.ranks, 'trunc', r.estimate.truncation_sse, 'bytes', len(r.container))
" >> gpurun_out/oz_diag.log 2>&1
echo done
