"""Inputs of the data_io fixture (shared by make_golden.py and the tests)."""

XC_GOOD = (
    "4 10 6\r\n"
    "0,5 1:0.5 3:-2.25 9:1e-3\r\n"
    " 2:1.0\n"
    "3\n"
    "1,2,4 0:0.0 7:3.5\n"
    "\n\n"
)
XC_BAD = {
    "empty": "",
    "header_fields": "3 4\n",
    "header_int": "3 x 4\n",
    "header_pos": "0 4 4\n",
    "label_int": "1 4 4\nq 1:1.0\n",
    "label_range": "1 4 4\n9 1:1.0\n",
    "feat_in_labels": "1 4 4\n1:2.0\n",
    "feat_token": "1 4 4\n1 2\n",
    "feat_num": "1 4 4\n1 a:b\n",
    "feat_inf": "1 4 4\n1 2:inf\n",
    "feat_range": "1 4 4\n1 4:1.0\n",
    "too_many": "1 4 4\n1 2:1.0\n2 1:1.0\n",
    "too_few": "3 4 4\n1 2:1.0\n",
}

# a run config exercising every section (the CLI fixture)
CLI_TOML = """
[data]
train = "train.txt"
normalize = true
[model]
hidden = [64]
lsh = "simhash"
k = 5
l = 8
beta = 40
bucket_capacity = 32
[train]
epochs = 2
batch_size = 32
learning_rate = 0.002
n0 = 10
seed = 7
eval_every = 5
eval_subsample = 100
[bench]
bench_sizes = [100, 1000]
bench_neurons = 2000
"""
