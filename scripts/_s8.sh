timeout 900 python -m pytest tests/test_gpu_gap.py tests/test_gpu_variants.py -x -q -k "gap or schedule" > gpurun_out/s8_tests.log 2>&1
timeout 900 python scripts/ab.py C3,C4,C5 2 'base:' 'ce4:AB_OPTS={"check_every":4}' 'ce8:AB_OPTS={"check_every":8}' 'relist:CG_RELIST=1' 'ce8relist:CG_RELIST=1,AB_OPTS={"check_every":8}' 'gap16:AB_OPTS={"gap_every":16}' 'ce8gap8:AB_OPTS={"check_every":8;"gap_every":8}' > gpurun_out/s8_ab.txt 2>&1
timeout 600 python scripts/slab_overhead.py C4 > gpurun_out/s8_slabs_colgr.jsonl 2>&1
timeout 600 env CG_RELABEL=bfs python scripts/slab_overhead.py C4 > gpurun_out/s8_slabs_bfs.jsonl 2>&1
