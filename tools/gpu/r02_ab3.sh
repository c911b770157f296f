cd $GRAFT_REPO_ROOT
O=gpurun_out/ab3; mkdir -p $O
for r in 1 2; do
timeout 300 python tools/m2l_ab.py /tmp/base.npy > $O/base_$r.log 2>&1
for V in og32 og64 og128; do FMM_LIB=paper_1106_5273_b200/build/variants/$V/libfmm_b200.so timeout 300 python tools/m2l_ab.py /tmp/$V.npy > $O/${V}_$r.log 2>&1; done
done
for V in og32 og64 og128; do python -c "
import numpy as np; a=np.load('/tmp/base.npy'); b=np.load('/tmp/$V.npy')
print('$V rel diff', float(np.linalg.norm(a-b)/np.linalg.norm(a)))" >> $O/diff.log 2>&1; done
