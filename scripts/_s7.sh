timeout 1500 python scripts/ab.py C3,C4,C5 4 'base:' 'ce4:AB_OPTS={"check_every":4}' 'ce6:AB_OPTS={"check_every":6}' 'ce12:AB_OPTS={"check_every":12}' 'b05:CG_GR_BETA=0.5' 'b07:CG_GR_BETA=0.7' 'b15:CG_GR_BETA=1.5' 'ce4b05:CG_GR_BETA=0.5,AB_OPTS={"check_every":4}' 'base2:' > gpurun_out/ab_knobs_trunc.txt 2>&1
cat gpurun_out/ab_knobs_trunc.txt
