cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "test_mono_path_matches_reference_goldens" 2>&1 | tail -4
timeout 600 python -m pytest tests -m gpu -q -x -k "test_mono_eval_matches_reference or test_mono_path_matches_reference_goldens" 2>&1 | tail -4
compute-sanitizer --tool memcheck python tools/gpu/dbg_dedup.py c2_surface_d3_xmem_t 2>&1 | tail -20
