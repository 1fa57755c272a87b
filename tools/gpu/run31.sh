set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "imag_health or eval_batch" > gpurun_out/pytest31.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest31.log
python -c "
import paper_2604_01059_b200 as zx
for n in ('c2_surface_d3_xmem_t','surface_d3_xmem_9t','surface_d3_xmem_rz5','c4_color_d5_rz3'):
    cs = zx.CompiledSampler.load('tests/golden/%s.zxs' % n); print(n, zx.imag_health(cs, 4096).round(6).tolist())
cs = zx.CompiledSampler.load('data/c3_cultivation_proxy.zxs.gz'); print('cultivation', zx.imag_health(cs, 256).tolist())
" 2>&1 | tee gpurun_out/imag31.txt
