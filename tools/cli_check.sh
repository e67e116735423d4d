# CLI on a B200 (run under gpurun): the GPU CLI tests, then one 8-GPU BERT sweep through the
# product binary (device engine) and through the same program on the reference CPU engine,
# timed, with the two output trees compared byte for byte.
set -x
TIMEFORMAT="real %R s"
mkdir -p gpurun_out/cli/dev gpurun_out/cli/ref
#python -m pytest tests/test_cli.py -m gpu -q > gpurun_out/cli/pytest.log 2>&1
nproc > gpurun_out/cli/nproc.txt
( cd gpurun_out/cli/dev && time ../../../paper_2202_13481_b200/msv sweep ../../../examples/sweep_bert_8gpu.json --out o ) > gpurun_out/cli/dev.log 2>&1
( cd gpurun_out/cli/ref && time ../../../oracle/_ref/msv_cli_ref sweep ../../../examples/sweep_bert_8gpu.json --out o ) > gpurun_out/cli/ref.log 2>&1
diff -r gpurun_out/cli/dev/o gpurun_out/cli/ref/o > gpurun_out/cli/diff.txt 2>&1 && echo IDENTICAL >> gpurun_out/cli/diff.txt
tail -3 gpurun_out/cli/pytest.log; grep -h "^real" gpurun_out/cli/dev.log gpurun_out/cli/ref.log; cat gpurun_out/cli/diff.txt | tail -3
