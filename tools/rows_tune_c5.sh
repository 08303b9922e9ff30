for r in 128 256; do
python - <<PY >> gpurun_out/t54.txt 2>&1
import sys; sys.argv=['x']
import sacd_inputs as SI, time
from paper_2003_03572_b200.sacd import Sacd
cfg=SI.CONFIGS['c5']
c,v=SI.make_tensor(cfg, device='cuda')
ref=None
for var in (2,0):
    g=Sacd(c,v,cfg.dims,$r,cfg.seed,rows_variant=var,profile=True)
    g.iterate(3); g.sync(); p=g.profile_read(); f=g.fit()[0]
    print('c5 R=$r rows variant',var,'rows ms/sweep %.3f'%(p['rows'][0]/3),'mttkrp %.3f'%(p['mttkrp'][0]/3), 'f',f, 'same' if ref is None or abs(f-ref)<=1e-9*abs(ref) else 'DIFF')
    ref=f; g.close()
PY
done
