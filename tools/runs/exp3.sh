mkdir -p gpurun_out/prof
cat > /tmp/chain_once.py <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np, torch, paper_2502_03000_b200 as lm
rng=np.random.default_rng(0)
X,Y,Z=(lm.DenseMatrix(np.asfortranarray(rng.uniform(-1,1,s))) for s in ((8000,100),(100,8000),(8000,100)))
for _ in range(3): lm.evaluate(X*Y*Z)
torch.cuda.synchronize()
PY
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:gemm_chain -s 2 -c 1 -o gpurun_out/prof/r02_chain -f python /tmp/chain_once.py > gpurun_out/prof/r02_chain.log 2>&1; echo rc=$?
