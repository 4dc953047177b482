#!/bin/bash
# ncu --set full captures of the HBM-bound checksum kernels and the QR panel
# (one GPU; summaries go to profiles/ after reading them here).
# usage: tools/gpu/prof_abft.sh TAG
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
# LU N=32768: the first encode (one read of the 32512^2 region) + two verify launches
timeout 900 $NCU -k regex:blocksum_kernel -c 1 -o gpurun_out/prof_blocksum_lu_$TAG \
  python bench.py --profile-only > gpurun_out/prof_blocksum_lu_$TAG.log 2>&1; echo "blocksum lu rc=$?"
timeout 900 $NCU -k regex:verify_kernel -c 2 -o gpurun_out/prof_verify_lu_$TAG \
  python bench.py --profile-only > gpurun_out/prof_verify_lu_$TAG.log 2>&1; echo "verify lu rc=$?"
# Cholesky N=32768: panel-column encodes (blocksum over (n-p) x b)
timeout 900 $NCU -k regex:blocksum_kernel -s 4 -c 2 -o gpurun_out/prof_blocksum_chol_$TAG \
  python bench.py --kind cholesky --profile-only > gpurun_out/prof_blocksum_chol_$TAG.log 2>&1; echo "blocksum chol rc=$?"
# QR N=32768: the first Householder panel (nk = 32768)
timeout 900 $NCU -k regex:qr_panel -c 1 -o gpurun_out/prof_qrpanel_$TAG \
  python bench.py --kind qr --profile-only > gpurun_out/prof_qrpanel_$TAG.log 2>&1; echo "qr panel rc=$?"
