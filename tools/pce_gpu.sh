python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests -m gpu -x -q -k "pce or block or camera or c2_query" 2>&1 | tail -4
python tools/fft_batch.py
python tools/pce_batch_once.py && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv python tools/pce_batch_once.py > gpurun_out/pce_ncu.csv 2>gpurun_out/pce_ncu.err
