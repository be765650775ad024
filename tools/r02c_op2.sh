python -c "import __graft_entry__ as g; g.build()" || exit 1
python tools/time_op.py C5 50; python tools/time_op.py C5 50
for mb in 6 8; do
  touch paper_1908_07071_b200/csrc/operator.cu
  LORPC_NVCC_EXTRA="-DLORPC_CG3_MINB=$mb" python -c "import __graft_entry__ as g; g.build()" || exit 1
  echo "MINB=$mb"; python tools/time_op.py C5 50; python tools/time_op.py C5 50
done
