# one call of the paper-space campaign: resume from the checkpoint committed under campaign/
# (copied into gpurun_out/, which is what comes back), sweep for the budget, checkpoint every chunk
mkdir -p gpurun_out/campaign
cp campaign/paper_fp16.npz* gpurun_out/campaign/ 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv >> gpurun_out/campaign/gpu.txt
python scripts/paper_campaign.py --ckpt gpurun_out/campaign/paper_fp16.npz --budget-s ${1:-5700}
