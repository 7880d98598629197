# batched drain of many short requests: which part of the batch path costs
S="python tools/small_requests.py --config c2 --tokens 128 --requests 32 --modes batch,batch1,merged"
$S
$S --variant 4 --threads 32 --stages 6 --ctas 48
$S --variant 2
