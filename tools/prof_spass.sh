# ncu --set full of the direct s-pass kernels (forced), one launch each
mkdir -p gpurun_out
export LFM_FWD_T=2 LFM_ADJ_T=2 LFM_FWD_SPLIT=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spass_fwd -c 1 -f -o gpurun_out/prof_spass \
  python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_1812_03358_b200 import lfm
from workloads import flame_volume, make_config, uniform_vector
cfg = make_config('128^3 two-camera')
plan = lfm.Plan(cfg, device=0); ws = plan.workspace()
x = torch.as_tensor(flame_volume(cfg['volume']), device='cuda:0').reshape(-1)
y = torch.empty(plan.infos[0]['n_pix'], device='cuda:0'); g = torch.empty_like(x)
lfm.A_forward(plan, 0, x, y, ws); lfm.A_adjoint(plan, 0, y, g, ws); torch.cuda.synchronize()
" > gpurun_out/prof_spass.log 2>&1; echo "NCU EXIT $?"; tail -3 gpurun_out/prof_spass.log
