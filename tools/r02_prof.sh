set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r02.csv python tools/one_step.py > gpurun_out/ncu1.log 2>&1
$NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/gemm_traffic_r02.csv python tools/one_step.py > gpurun_out/ncu2.log 2>&1
$NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k "regex:ln_|xent_|sgd_|embed_|qkv_grad|attn_rowdot|cast_|fold_|check_ids|colsum|flash" --clock-control none --csv --log-file gpurun_out/rowops_r02.csv python tools/one_step.py > gpurun_out/ncu3.log 2>&1
timeout 900 python bench.py --workload gpt --checkpointing --max-batch --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/gpt_maxb_train_ckpt.json 2> gpurun_out/gpt_maxb.err
timeout 600 python bench.py --workload bert --max-batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bert_maxb_train.json 2> gpurun_out/bert_maxb.err
