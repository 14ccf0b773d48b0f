/* C restatement of the reference hot path (see qtrain_oracle.c) */
#pragma once
